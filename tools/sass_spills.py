"""Spill (STL/LDL) sites of one kernel per CUDA source line: python tools/sass_spills.py <nvdisasm -g output> <kernel substring>
(profiling aid: run `cuobjdump -xelf all x.o; nvdisasm -g x.cubin > all.sass` first)."""
import re
import sys

text = open(sys.argv[1]).read().split("\n")
want = sys.argv[2]
inside = False
cur = None
out = {}
for l in text:
    if l.startswith(".text."):
        inside = want in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"\b(STL|LDL)(\.[0-9A-Z]+)*\b", l):
        out.setdefault(cur, 0)
        out[cur] += 1
for k, v in sorted(out.items(), key=lambda kv: str(kv[0])):
    print(k, v)
