"""Thread slots lost to divergence / predication per SASS instruction of an ncu
capture (source page): where the warp runs with few active threads.
usage: python tools/lost_slots.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out)
next(r)
h = next(r)
ia, isrc = h.index("Address"), h.index("Source")
ie, it = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
rows = []
for x in r:
    try:
        rows.append((x[ia], x[isrc].strip(), int(x[ie]), int(x[it])))
    except (ValueError, IndexError):
        continue
te = sum(e for *_, e, _ in rows)
tt = sum(t for *_, t in rows)
print(f"{te} warp instructions, {tt / te:.2f} threads each, {100 * (1 - tt / (32 * te)):.1f}% "
      "thread slots lost")
for a, src, e, t in sorted(rows, key=lambda x: -(32 * x[2] - x[3]))[:top]:
    print(f"{a[-5:]} {e:>10} {t / e:6.2f} thr  lost {32 * e - t:>11}  {src[:70]}")
