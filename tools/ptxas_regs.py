"""Registers / spills per k_eval instantiation from a ptxas -v log."""
import re
import sys

fn = None
for l in open(sys.argv[1]).read().splitlines():
    m = re.search(r"Compiling entry function '(\S+)'|Function properties for (\S+)", l)
    if m:
        fn = m.group(1) or m.group(2)
    m = re.search(r"Used (\d+) registers", l)
    if m and fn and "k_eval" in fn:
        k = re.search(r"k_evalI([df])Li(\d+)ELi(\d+)E", fn)
        print(f"{'f64' if k.group(1) == 'd' else 'f32'} fn={k.group(2):>2} vw={k.group(3)} regs={m.group(1)}")
