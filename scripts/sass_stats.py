"""Opcode histogram of one kernel in a cuobjdump -sass listing."""
import re
import sys
from collections import Counter

path, name = sys.argv[1], sys.argv[2]
lines = open(path).read().split("\n")
start = [i for i, l in enumerate(lines) if "Function : " in l and name in l][0]
end = next((i for i, l in enumerate(lines) if "Function :" in l and i > start), len(lines))
k = [l for l in lines[start:end] if re.search(r"/\*[0-9a-f]{4,6}\*/", l)]
c = Counter(re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", l).group(2) for l in k)
print(len(k), "instructions")
print(c.most_common(30))

# main loop: the largest backward branch
addr = lambda l: int(re.search(r"/\*([0-9a-f]{4,6})\*/", l).group(1), 16)
best = None
for l in k:
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", l)
    if m:
        a, b = addr(l), int(m.group(1), 16)
        if b < a and (best is None or a - b > best[0] - best[1]):
            best = (a, b)
if best:
    body = [l for l in k if best[1] <= addr(l) <= best[0]]
    cb = Counter(re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", l).group(2) for l in body)
    print(f"main loop {hex(best[1])}..{hex(best[0])}: {len(body)} instructions")
    print(cb.most_common(30))
