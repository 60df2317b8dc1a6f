"""Per-source-line hot spots from `ncu -i X --page source --csv --print-source cuda,sass`:
python profiles/srclines.py dump.csv [top]  -> lines ranked by stall samples."""
import csv
import sys

rows, cur_file = [], None
with open(sys.argv[1], newline="") as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "" or len(r) < 8:
            continue
        try:
            rows.append((cur_file, int(r[0]), r[1][:70], int(r[4] or 0), int(r[7] or 0)))
        except ValueError:
            pass
tot_s = sum(x[3] for x in rows) or 1
tot_i = sum(x[4] for x in rows) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total stall samples {tot_s}, warp instructions {tot_i:.3e}")
print("| file:line | samples % | inst % | source |\n|---|---|---|---|")
for fn, ln, src, s, i in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"| {fn}:{ln} | {100*s/tot_s:.1f} | {100*i/tot_i:.1f} | `{src.strip()}` |")
