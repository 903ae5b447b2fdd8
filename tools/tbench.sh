# quick C2 triplet + step timing: prints ms_per_step and the roofline.triplet fwd/bwd times
python bench.py --steps 20 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=d['roofline']['triplet']
print('step %.3f ms  fwd %.1f us  bwd %.1f us' % (d['ms_per_step'], t['fwd_us'], t['bwd_us']))"
