"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel name.

    python tools/launch_summary.py gpurun_out/r1_launches.csv [--last N] > profiles/r1_launches_summary.txt

--last N keeps only the last N launches (the final profiled step)."""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    seen, order = {}, []
    for r in rows:  # one row per launch (ID)
        if r["ID"] not in seen:
            seen[r["ID"]] = r
            order.append(r["ID"])
    launches = [seen[i] for i in order]
    if last:
        launches = launches[-last:]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in launches:
        name = r["Kernel Name"].split("(")[0][:90]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000 if unit in ("nsecond", "ns") else v * 1000 if unit in ("msecond", "ms") else v
        tot[name] += us
        cnt[name] += 1
    total = sum(tot.values())
    print(f"{len(launches)} launches, {total:.1f} us summed kernel time (ncu, serialised, cold-ish caches)")
    print(f"{'kernel':90s} {'n':>5s} {'total us':>10s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:90s} {cnt[k]:5d} {tot[k]:10.1f} {100 * tot[k] / total:6.1f}%")


if __name__ == "__main__":
    main()
