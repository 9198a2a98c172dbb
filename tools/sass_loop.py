"""Largest inner loop of a kernel in a cubin/.o: instruction mix (build-time check)."""
import re
import subprocess
import sys

obj, kernel = sys.argv[1], sys.argv[2]
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
start = txt.index("Function : " + kernel)
body = txt[start:]
nxt = body.find("Function : ", 10)
body = body[: nxt if nxt > 0 else None]
lines = [re.sub(r"\s+", " ", l.split(";")[0]) for l in body.split("\n") if "/*" in l and ";" in l]
addr = lambda l: int(re.search(r"/\*([0-9a-f]+)\*/", l).group(1), 16)  # noqa: E731
best = None
for l in lines:
    m = re.search(r"BRA (0x[0-9a-f]+)", l)
    if m and int(m.group(1), 16) < addr(l):
        t, a = int(m.group(1), 16), addr(l)
        blk = [x for x in lines if t <= addr(x) <= a]
        key = sys.argv[3] if len(sys.argv) > 3 else "VIMNMX"
        # innermost loop doing the work: fewest instructions with >= 8 `key` ops
        if sum(key in x for x in blk) >= 8 and (best is None or len(blk) < len(best)):
            best = blk
ops = {}
for x in best:
    op = x.split("*/")[1].strip().split(" ")[0]
    op = op if not op.startswith("@") else x.split("*/")[1].strip().split(" ")[1]
    ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
print(len(best), "instructions:", dict(sorted(ops.items(), key=lambda kv: -kv[1])))
