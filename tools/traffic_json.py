"""Write profiles/r1_traffic.json (DRAM bytes per launch) from ncu --set full reports.

    python tools/traffic_json.py KEY=REPORT[:KERNEL_SUBSTRING] ... --edges E --triplets T --dg D
Each KEY sums dram__bytes_read/write over the report's launches whose name contains
KERNEL_SUBSTRING (all launches if omitted)."""
import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return int(float(v.replace(",", "")) * scale)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--edges", type=int, required=True)
    ap.add_argument("--triplets", type=int, required=True)
    ap.add_argument("--dg", type=int, required=True)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r2_traffic.json"))
    a = ap.parse_args()
    res = {"_comment": "DRAM bytes per launch from ncu --set full captures (tools/traffic_json.py; "
                       "summaries in profiles/r2_*_ncu.txt)",
           "workload": {"edges": a.edges, "triplets": a.triplets, "dg": a.dg}}
    for spec in a.specs:
        key, rest = spec.split("=", 1)
        rd = wr = 0
        names, reps = [], []
        for part in rest.split("+"):  # several reports (e.g. the two backward kernels) sum
            rep, _, sub = part.partition(":")
            reps.append(Path(rep).name)
            out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
            rows = list(csv.reader(io.StringIO(out)))
            hdr, units = rows[0], rows[1]
            u = dict(zip(hdr, units))
            for row in rows[2:]:
                d = dict(zip(hdr, row))
                if sub and sub not in d.get("Kernel Name", ""):
                    continue
                names.append(d.get("Kernel Name", "")[:80])
                rd += to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
                wr += to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        res[key] = {"kernels": names, "dram_read": rd, "dram_write": wr, "reports": reps}
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
