"""Summarise an ncu `--page source --csv --print-source cuda,sass` export by
CUDA source line: warp-stall samples and executed instructions (top N)."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur, hdr, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        stall = int(r[4]); inst = int(r[7]); thr = int(r[8])
    except ValueError:
        continue
    out.append((stall, inst, thr, cur, r[0], r[1].strip()[:90]))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for s, i, t, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% stall {100*i/tot_i:5.1f}% inst  thr/inst {t/max(i,1):5.1f}  {f}:{ln}  {src}")
