"""Per-source-line executed warp instructions and stall samples of one kernel
in an ncu report (source page, cuda+sass).  usage: ncu_inst.py REP KERNEL [TOP]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
ex = collections.Counter()
smp = collections.Counter()
src = {}
cur = None
fname = "?"
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, r[0])
        src[cur] = r[1].strip()[:90]
    try:
        ex[cur] += int(r[7])
        smp[cur] += int(r[4])
    except ValueError:
        pass
te, ts = sum(ex.values()) or 1, sum(smp.values()) or 1
print(f"total warp instructions {te}")
for key, v in ex.most_common(top):
    print(f"{100.0 * v / te:5.1f}% inst {100.0 * smp[key] / ts:5.1f}% smp {key[0]}:{key[1]}  {src.get(key, '')}")
