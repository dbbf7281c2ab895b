"""Per-source-line warp-stall samples from an ncu report's source page
(ncu -i REP --page source --csv --print-source cuda,sass): the lines a
kernel spends its time on.  usage: ncu_lines.py REP KERNEL_REGEX [TOP]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
acc = collections.Counter()
src = {}
cur = None
fname = "?"
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, r[0])
        src[cur] = r[1].strip()[:100]
    try:
        acc[cur] += int(r[4])
    except ValueError:
        pass
tot = sum(acc.values()) or 1
for key, v in acc.most_common(top):
    print(f"{100.0 * v / tot:5.1f}% {key[0]}:{key[1]}  {src.get(key, '')}")
