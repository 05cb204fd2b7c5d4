"""Per-kernel counts of the instructions that show the B200 programming model
in the built library (cuobjdump -sass): tcgen05 MMAs (UTC*MMA), TMA
(UTMALDG / UTMASTG / UBLKCP / UTMAREDG), TMEM loads / stores (LDTM / STTM),
mbarrier ops (SYNCS), and the legacy tensor path (HMMA, must be 0).
    python tools/sass_summary.py > profiles/r01/sass_summary.md"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2605_10905_b200/libmimw_b200.so"
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "UBLKRED", "LDTM", "STTM",
        "UTCCP", "SYNCS", "MUFU.EX2", "HMMA"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
cur = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m:
        op = m.group(1)
        for k in KEYS:
            if op.startswith(k):
                counts[cur][k] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = d.replace("(anonymous namespace)::", "")
    d = re.sub(r"\(.*", "", d).replace("mimw::", "")
    return d[:90]


print("| kernel | " + " | ".join(KEYS) + " |")
print("|---|" + "---|" * len(KEYS))
for fn, c in counts.items():
    if not any(c.values()):
        continue
    print(f"| `{short(fn)}` | " + " | ".join(str(c[k]) for k in KEYS) + " |")
