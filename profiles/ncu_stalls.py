"""Per-source-line warp-stall breakdown from an ncu source-page CSV export
(`ncu -i rep --page source --csv --print-source cuda,sass [-k kernel]`)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur = hdr = None
out, tot = [], {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 50 or r[2] != "-":
        continue
    st = {hdr[i]: int(r[i]) for i in range(32, 49) if r[i].isdigit()}
    for k, v in st.items():
        tot[k] = tot.get(k, 0) + v
    out.append((int(r[4]), cur, r[0], r[1].strip()[:70], st, int(r[7])))
T = sum(tot.values()) or 1
print({k.replace("stall_", ""): round(100 * v / T, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
print("warp instructions", round(sum(o[5] for o in out) / 1e6), "M")
for s, f, l, src, st, inst in sorted(out, reverse=True)[:top]:
    t3 = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{100*s/T:5.1f}% {f}:{l} inst={inst/1e6:.0f}M "
          f"{[(k.replace('stall_', ''), round(100*v/max(s, 1))) for k, v in t3]} | {src}")
