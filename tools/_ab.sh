cp paper_2203_09697_b200/libegn_b200.so /tmp/orig.so
for rep in 1 2; do
for d in build/var_old build/var_new; do
  cp $d/libegn_b200.so paper_2203_09697_b200/libegn_b200.so
  python bench.py --no-cpu-baseline --no-kernel-timing --steps 200 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$d', round(d['ms_per_step'],4), d['e2e']['ms_per_step'])"
done
done
cp /tmp/orig.so paper_2203_09697_b200/libegn_b200.so
