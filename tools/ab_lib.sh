#!/bin/bash
# Same-box A/B of two library builds: tools/ab_lib.sh [steps]
# (A = paper_2203_09697_b200/libegn_b200.so, B = paper_2203_09697_b200/libegn_b200_alt.so)
steps=${1:-50}
for rep in 1 2; do
  for lib in libegn_b200.so libegn_b200_alt.so; do
    EGN_LIB=paper_2203_09697_b200/$lib python bench.py --steps "$steps" --warmup 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'], d['e2e']['ms_per_step'])"
  done
done
