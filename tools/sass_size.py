"""Per-kernel SASS size of a cubin/.so dump (cuobjdump -sass > file)."""
import collections
import re
import sys

cnt = collections.Counter()
name = None
for line in open(sys.argv[1]):
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = m.group(1)
        continue
    if name and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        cnt[name] += 1
for n, c in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    print(f"{c:7d} instr {c * 16 / 1024:7.1f} KB  {n[:90]}")
