"""Dynamic opcode mix from an ncu report's SASS source page (per element)."""
import csv, io, re, subprocess, sys, collections
path, n = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iT, iP, iW = hdr.index("Source"), hdr.index("Thread Instructions Executed"), \
    hdr.index("Predicated-On Thread Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
c, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iT:
        continue
    s = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
    op = s.split()[0] if s else "?"
    t = float(r[iP] or 0)
    c[op] += t
    stall[op] += float(r[iW] or 0)
    tot += t
print(f"thread instructions per element: {tot / n:.1f}")
fp = {k: v for k, v in c.items() if k.split('.')[0] in ('DADD', 'DMUL', 'DFMA', 'FADD', 'FMUL', 'FFMA')}
print("FP per element:", {k: round(v / n, 1) for k, v in sorted(fp.items())}, "sum", round(sum(fp.values()) / n, 1))
print("top ops per element:", ", ".join(f"{k} {v / n:.1f}" for k, v in c.most_common(30)))
st = sum(stall.values()) or 1
print("stall samples by op:", ", ".join(f"{k} {v / st:.0%}" for k, v in stall.most_common(10)))
