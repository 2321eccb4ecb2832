"""Top source lines by warp-stall samples from an ncu report, mapping SASS
offsets to file:line with nvdisasm line info of the given cubin/.so.
python tools/ncu_hot.py report.ncu-rep lib.so [kernel] [N]"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib = sys.argv[1], sys.argv[2]
kern = sys.argv[3] if len(sys.argv) > 3 else "rapdb_solver_kernel"
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
iS = h.index("Warp Stall Sampling (All Samples)")
samples = []
for r in rows[1:]:
    try:
        samples.append((int(r[0], 16), int(float(r[iS] or 0)), r[1].strip()))
    except (ValueError, IndexError):
        continue
base = samples[0][0]
# offset -> (file, line) from nvdisasm -gi
tmp = tempfile.mkdtemp()
if lib.endswith(".cubin"):
    cub = lib
else:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-gi", "-fun", kern, cub], capture_output=True, text=True).stdout
if not dis.strip():
    dis = subprocess.run(["nvdisasm", "-gi", cub], capture_output=True, text=True).stdout
loc = {}
cur = None
infun = False
for l in dis.splitlines():
    if re.match(r"\s*\.text\.", l) or l.startswith(".text."):
        infun = kern in l
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur is not None:
        loc.setdefault(int(m.group(1), 16), cur)
agg = {}
tot = 0
for addr, v, src in samples:
    tot += v
    key = loc.get(addr - base, ("?", 0))
    agg[key] = agg.get(key, 0) + v
print("total samples", tot)
for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:N]:
    print(f"{v:7d} {100.0 * v / max(tot, 1):5.1f}%  {key[0]}:{key[1]}")
