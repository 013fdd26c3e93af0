"""Summarise a compute-sanitizer racecheck log: hazards grouped by (kind, kernel, source line)."""
import collections
import re
import sys

cnt = collections.Counter()
kind = None
for line in open(sys.argv[1], errors="replace"):
    m = re.search(r"(Error|Warning): \(?([^)]*?)\)? ?(Potential )?(\w+) hazard", line)
    if m:
        kind = (m.group(1), m.group(4))
        continue
    m = re.search(r"(Read|Write) Thread .* at (?:void )?([\w:<>(), ]+?)\(.*? in ([\w.]+:\d+)", line)
    if m and kind:
        cnt[(kind, m.group(1), m.group(2).split("(")[0][-60:], m.group(3))] += 1
for k, v in cnt.most_common(40):
    print(v, *k)
print("total hazard lines", sum(cnt.values()))
