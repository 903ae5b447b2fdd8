#!/bin/bash
# A/B a runtime knob on one box: tools/ab_env.sh VAR "v1 v2 ..." [steps]
# prints ms_per_step and e2e for each value, interleaved twice
var=$1; vals=$2; steps=${3:-50}
for rep in 1 2; do
  for v in $vals; do
    env "$var=$v" python bench.py --steps "$steps" --warmup 5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', d['ms_per_step'], d['e2e']['value'])"
  done
done
