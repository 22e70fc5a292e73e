"""Where a kernel spills: count STL/LDL per source line (nvdisasm -g).
usage: python tools/spills.py OBJ.o MANGLED_KERNEL"""
import collections, os, re, subprocess, sys, tempfile
obj, fn = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    s = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True, text=True).stdout
st = s.index(f"//--------------------- .text.{fn} ")
nx = s.find("//--------------------- ", st + 10)
cur, c = None, collections.Counter()
for line in s[st:nx if nx > 0 else len(s)].splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    for op in ("STL", "LDL"):
        if re.search(r"\b" + op + r"\b", line):
            c[(cur, op)] += 1
for k, v in sorted(c.items(), key=lambda kv: -kv[1])[:40]:
    print(v, k)
