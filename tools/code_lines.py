"""Static SASS instruction count per source line inside one function of an
`nvdisasm -g` listing (cubin compiled with -lineinfo).
Usage: python tools/code_lines.py listing.nvd <function-substring> [top]"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
pat = sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
inside = False
cur = None
cnt = Counter()
for ln in lines:
    s = ln.strip()
    if re.match(r"^\$?\$?[\w$.]+:\s*$", s) and not s.startswith(".L"):
        inside = pat in s
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', s)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", s):
        cnt[cur] += 1
tot = sum(cnt.values())
print(f"{pat}: {tot} instructions ({16 * tot / 1024:.1f} KB)")
for (k, v) in cnt.most_common(top):
    print(f"  {v:5d}  {k}")
