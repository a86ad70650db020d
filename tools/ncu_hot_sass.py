"""Top SASS instructions by warp-stall samples for each kernel of an ncu report
(run here, no GPU needed):  python tools/ncu_hot_sass.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
parts = raw.split('"Kernel Name",')[1:]
for part in parts:
    lines = part.splitlines()
    name = lines[0].strip().strip(",").strip('"')
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    ia = hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[1:] if len(r) > ia and r[ia] not in ("", "-")]
    tot = sum(float(r[ia]) for r in body) or 1.0
    print(f"== {name[:110]}  ({len(body)} instructions, {tot:.0f} samples)")
    for r in sorted(body, key=lambda r: -float(r[ia]))[:top]:
        print(f"  {100 * float(r[ia]) / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:100]}")
