"""Per-kernel histogram of the Blackwell-native SASS in libxknn.so (no GPU needed):
UTCHMMA/UTCQMMA (tcgen05.mma), UTMALDG/UTMASTG/UBLKCP (TMA), LDTM/STTM (TMEM), UTCBAR (tcgen05
commit), SYNCS (mbarriers), MUFU.EX2.

    python tools/sass_histogram.py > profiles/r02/sass_histogram.txt
"""
import collections
import re
import subprocess
import sys
import os

LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2102_06025_b200",
    "libxknn.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCBAR",
        "SYNCS", "MUFU.EX2", "HMMA", "LDG", "STG"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
func, hist = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        func = m.group(1)
        hist[func] = collections.Counter()
        continue
    if func is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if not m:
        continue
    op = m.group(2)
    for k in KEYS:
        if op == k or op.startswith(k + ".") or (k == "MUFU.EX2" and op.startswith("MUFU.EX2")):
            hist[func][k] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


names = list(hist)
pretty = demangle(names)
print(f"# {LIB}\n# kernel: " + " ".join(KEYS))
for n, p in zip(names, pretty):
    h = hist[n]
    if not any(h[k] for k in KEYS[:8]):
        continue
    q = p.replace("(anonymous namespace)::", "").replace("xknn::", "")
    q = re.sub(r"^void ", "", q)
    short = q.split("(")[0]
    print(f"{short[:60]:60s} " + " ".join(f"{k}={h[k]}" for k in KEYS if h[k]))
