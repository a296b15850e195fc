"""Executed instructions per source line (and per opcode on that line) from an
ncu report's SASS page, joined with nvdisasm line info of the same build.
usage: python tools/ncu_lines.py report.ncu-rep <mangled-kernel> <elements> [top]
The library in paper_1502_05216_b200/lib must be the build that was profiled."""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, kern, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
so = "paper_1502_05216_b200/lib/libtwofold_b200.so"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith("tf_kernels")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout
loc, cur, inside = {}, None, False
for ln in dis.splitlines():
    if ln.startswith(kern + ":"):
        inside = True
        continue
    if inside and re.match(r"^\S+:$", ln) and not ln.startswith(".text." + kern):
        if not ln.startswith(".L"):
            break
    if not inside:
        continue
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
    if m:
        loc[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iA, iS, iP, iW = (hdr.index("Address"), hdr.index("Source"),
                  hdr.index("Predicated-On Thread Instructions Executed"),
                  hdr.index("Warp Stall Sampling (All Samples)"))
base = None
per_line, per_op, stall = collections.Counter(), collections.defaultdict(collections.Counter), collections.Counter()
for r in rows[2:]:
    if len(r) <= iP or not r[iA].startswith("0x"):
        continue
    a = int(r[iA], 16)
    base = a if base is None else base
    key = loc.get(a - base, ("?", 0))
    s = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
    op = s.split()[0] if s else "?"
    t = float(r[iP] or 0) / n
    per_line[key] += t
    per_op[key][op] += t
    stall[key] += float(r[iW] or 0)
tot, st = sum(per_line.values()), sum(stall.values()) or 1
print(f"{tot:.1f} thread instructions per element")
for key, v in per_line.most_common(top):
    ops = ", ".join(f"{o} {c:.1f}" for o, c in per_op[key].most_common(6))
    print(f"{key[0]}:{key[1]:<5d} {v:6.1f}  stall {stall[key] / st:5.1%}  {ops}")
