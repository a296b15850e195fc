"""Executed SASS opcode mix of an ncu report (source page, per-instruction
'Instructions Executed' x threads), normalised per element."""
import collections
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hi]
si, ti = hdr.index("Source"), hdr.index("Thread Instructions Executed")
c = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= ti:
        continue
    src = r[si].strip()
    src = src.split(";")[0]
    toks = src.split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    try:
        c[op] += float(r[ti].replace(",", ""))
    except ValueError:
        pass
tot = sum(c.values())
print(f"thread instructions per element: {tot / n:.1f}")
print(", ".join(f"{k} {v / n:.1f}" for k, v in c.most_common(40)))
