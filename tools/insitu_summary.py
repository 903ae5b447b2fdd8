"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of tools/profile_step.py --plain --steps 1:
the last step's launches grouped by kernel."""
import collections
import csv
import sys


def main(path, nsteps=4):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ker = {}
    for r in rows[1:]:
        if r[im] == "gpu__time_duration.sum":
            ker[int(r[iid])] = (r[ik], float(r[iv]))
    items = [ker[k] for k in sorted(ker)]
    step = items[-(len(items) // nsteps):]
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for nm, t in step:
        key = nm.split("(")[0][:70]
        tot[key] += t
        cnt[key] += 1
    print(f"{path}: {len(step)} launches, device time {sum(tot.values()) / 1e3:.1f} us")
    for nm, t in sorted(tot.items(), key=lambda kv: -kv[1])[:14]:
        print(f"  {nm:70s} {cnt[nm]:4d} {t / 1e3:8.1f} us {t / cnt[nm] / 1e3:7.1f} us/call")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
