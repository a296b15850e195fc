"""Opcode mix of a kernel's SASS (whole kernel and the hottest loop body).
usage: python tools/sass_mix.py <mangled-kernel-name-substring>"""
import re, subprocess, sys, collections
so = "paper_1502_05216_b200/lib/libtwofold_b200.so"
txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
want = sys.argv[1]
cur, lines = None, []
for ln in txt.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    if cur and want in cur:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            lines.append((int(m.group(1), 16), m.group(2).strip()))
def op(s):
    s = re.sub(r"^@!?U?P\w+\s+", "", s)
    return s.split()[0]
# main loop = the backward branch spanning the first LDGSTS (the streaming loop)
ld = [a for a, s in lines if "LDGSTS" in s]
loops = []
for a, s in lines:
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", s)
    if m and m.group(1):
        t = int(m.group(1), 16)
        if t < a:
            loops.append((t, a))
outer = [l for l in loops if ld and l[0] <= ld[-1] <= l[1]]
main = max(outer, key=lambda l: l[1] - l[0]) if outer else None
for name, rng in (("kernel", None), ("main loop", main)):
    c = collections.Counter(op(s) for a, s in lines if rng is None or rng[0] <= a <= rng[1])
    tot = sum(c.values())
    fp64 = sum(v for k, v in c.items() if k.split(".")[0] in ("DADD", "DMUL", "DFMA"))
    print(f"== {name} {rng}: {tot} instr, FP64 {fp64}")
    print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common(28)))
