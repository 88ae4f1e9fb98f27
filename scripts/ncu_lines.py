"""Per-source-line warp-stall samples of one file from an ncu report (cuda,sass source view):
    python scripts/ncu_lines.py report.ncu-rep file_substring [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr = None, None
acc = defaultdict(lambda: [0, 0, ""])
total = 0
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 5 or not row[0]:
        continue
    try:
        s = int(row[4] or 0)
    except ValueError:
        continue
    total += s
    if cur and want in cur:
        a = acc[int(row[0])]
        a[0] += s
        try:
            a[1] += int(row[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            pass
        a[2] = row[1][:90]
tot_file = sum(v[0] for v in acc.values())
print(f"total samples {total}; {want}: {tot_file} ({100.0 * tot_file / max(1, total):.1f}%)")
for ln, (sm, ins, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {sm:7d} {100.0 * sm / max(1, total):5.2f}% inst {ins:10d}  {src.strip()}")
