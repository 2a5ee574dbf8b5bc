"""Map an ncu SASS source page (--page source --csv --print-source sass) to
CUDA source lines with nvdisasm -g of the same cubin (developer tool):

    python tools/ncu_srcmap.py CUBIN MANGLED_NAME SASS_CSV UNITS [SRC_DIR]

UNITS divides the thread-instruction counts (e.g. vehicles x steps).
"""
import csv, os, re, sys, collections, subprocess
cubin, fun, sass_csv, nveh = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
srcdir = sys.argv[5] if len(sys.argv) > 5 else os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2305_16510_b200", "csrc")
dis = subprocess.run(["nvdisasm", "-g", "-c", "-fun", fun, cubin], capture_output=True, text=True).stdout
if not dis.strip():
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    a = dis.index(".text." + fun + ":")
    b = dis.find("//---------------------", a)
    dis = dis[a:b if b > 0 else None]
cur = None; off2line = {}
for line in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', line)
    if m: off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]; ti = hdr.index("Thread Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > ti]
base = int(data[0][0], 16)
agg = collections.Counter(); st = collections.Counter(); tot = 0; stot = 0
for r in data:
    off = int(r[0], 16) - base
    key = off2line.get(off, ("?", 0))
    t = int(r[ti]); agg[key] += t; tot += t; st[key] += int(r[si]); stot += int(r[si])
print("instructions mapped:", len(data), "of", len(off2line), " total thread-inst/vehicle", tot / nveh)
src = {}
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:int(os.environ.get("SRCMAP_TOP", "45"))]:
    if f not in src:
        try: src[f] = open(os.path.join(srcdir, f)).read().splitlines()
        except Exception: src[f] = []
    txt = src[f][l - 1].strip()[:70] if 0 < l <= len(src[f]) else ""
    print(f"{v / nveh:7.1f} inst/veh  stall {100 * st[(f, l)] / stot:5.1f}%  {f}:{l}  {txt}")
