"""Instruction count per source line of one kernel (nvdisasm -g output), for a line range.
usage: sass_lines.py <file.sass> <function-substring> <src-file-substring> <lo> <hi>"""
import re, sys, collections
path, fn, src, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
inside = False
cur = None
cnt = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for line in open(path):
    if line.startswith("//--------------------- .text."):
        inside = fn in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = int(m.group(2)) if src in m.group(1) else None
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur is not None and lo <= cur <= hi:
        cnt[cur] += 1
        ops[cur][m.group(2)] += 1
tot = sum(cnt.values())
print("total", tot)
for l in sorted(cnt):
    print(l, cnt[l], dict(ops[l].most_common(6)))
