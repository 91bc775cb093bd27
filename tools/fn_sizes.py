"""Static size of every function in an nvdisasm listing (KB of SASS)."""
import re
import sys

cur, sizes = None, {}
for line in open(sys.argv[1]):
    s = line.strip()
    m = re.match(r"^(\$?\$?[\w$.]+):\s*$", s)
    if m and not s.startswith(".L"):
        cur = re.sub(r"_ZN49_INTERNAL_\w+?4slse", "", m.group(1).split("$")[-1])[:70]
        continue
    if cur and re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", s):
        sizes[cur] = sizes.get(cur, 0) + 1
tot = sum(sizes.values())
print(f"total {16 * tot / 1024:.0f} KB")
for k, v in sorted(sizes.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{16 * v / 1024:7.1f} KB  {k}")
