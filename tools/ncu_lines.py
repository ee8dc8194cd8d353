"""Per-source-line instruction / stall-sample shares from an ncu report
(--page source --print-source cuda,sass).  Usage: ncu_lines.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = None
hdr = None
recs = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":  # cuda-line rows carry '-' in the SASS address column
        try:
            recs.append((cur_file, int(r[0]), r[1].strip()[:80], int(r[7] or 0), int(r[4] or 0)))
        except ValueError:
            pass
ti = sum(x[3] for x in recs) or 1
ts = sum(x[4] for x in recs) or 1
print(f"instructions {ti:,}  stall samples {ts:,}")
for f, ln, src, ie, st in sorted(recs, key=lambda x: -(x[3] / ti + x[4] / ts))[:top]:
    print(f"{ie / ti * 100:5.1f}% inst {st / ts * 100:5.1f}% stall  {f}:{ln}  {src}")
