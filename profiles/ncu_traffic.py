"""Per-launch DRAM traffic of one kernel from an `ncu --set full` report:
writes profiles/traffic.json, which bench.py reports as roofline.traffic.

  python profiles/ncu_traffic.py <report.ncu-rep> <kernel-substring> [tag]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    tag = sys.argv[3] if len(sys.argv) > 3 else Path(rep).stem
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    rd, wr, du = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("gpu__time_duration.sum")
    best = None
    for r in rows[2:]:
        if pat not in r[ki]:
            continue
        t = float(r[rd]) * UNITS[units[rd]] + float(r[wr]) * UNITS[units[wr]]
        dur = float(r[du])
        if best is None or dur > best[2]:  # the full-size launch (not a tiny finish pass)
            best = (t, r[ki], dur)
    if best is None:
        raise SystemExit(f"no launch of {pat!r} in {rep}")
    d = {"kernel": best[1][:160], "traffic_bytes": best[0], "duration_us_ncu": best[2], "source": tag}
    Path(__file__).with_name("traffic.json").write_text(json.dumps(d, indent=1) + "\n")
    print(d)


if __name__ == "__main__":
    main()
