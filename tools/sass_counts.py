"""SASS evidence: tcgen05 / TMA / TMEM instruction counts and code size per kernel of libstree.so.
    python tools/sass_counts.py > profiles/rNN/sass_tcgen05_tma.txt"""
import collections
import os
import re
import subprocess

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2505_14969_b200", "libstree.so")
OPS = ("UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR", "SYNCS", "ELECT", "MUFU")

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
print("cuobjdump -sass paper_2505_14969_b200/libstree.so: tcgen05 / TMA / TMEM instruction counts and code size per kernel")
print("(UTCHMMA = tcgen05.mma kind::f16/tf32, UTMALDG/UTMASTG = TMA tensor load/store, UBLKCP = 1-D bulk copy,")
print(" LDTM/STTM = tcgen05.ld/st, UTCBAR = tcgen05.commit, SYNCS = mbarrier ops, ELECT = elect.sync, MUFU = SFU)")
name, counts, nins = None, collections.Counter(), 0


def flush():
    if name:
        print(f"{name} {nins * 16} B SASS")
        print("   ", dict(sorted(counts.items())))


for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        flush()
        name, counts, nins = m.group(1), collections.Counter(), 0
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9]+)", line)
    if m and name:
        nins += 1
        op = m.group(1)
        if op in OPS:
            counts[op] += 1
flush()
