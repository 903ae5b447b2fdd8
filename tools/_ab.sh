cp paper_2203_09697_b200/libegn_b200.so /tmp/orig.so
for d in build/var_A build/var_B build/var_AB; do
  cp $d/libegn_b200.so paper_2203_09697_b200/libegn_b200.so
  echo "== $d"; python tools/debug_precision.py 2>&1 | grep "gemnet-style tc=True" | cut -c1-120
done
for r in 1 2; do
for d in build/var_A build/var_B build/var_AB; do
  cp $d/libegn_b200.so paper_2203_09697_b200/libegn_b200.so
  python bench.py --no-cpu-baseline --no-kernel-timing --steps 200 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$d', round(d['ms_per_step'],4))"
done
done
cp /tmp/orig.so paper_2203_09697_b200/libegn_b200.so
