"""Timeline of CTA 0 of the attention kernel (debug aid; build with
MIMW_NVCC_EXTRA=-DMIMW_FA_EVENTS).  Prints, per KV step of the first work
item, when the MMA warp issued S0/PV0/S1/PV1 and when the softmax warps of the
two Q tiles saw S, had it loaded, had PV done and published P (cycles
relative to the step's S0 issue)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

bh, s = 128, 8192
emu = int(sys.argv[1]) if len(sys.argv) > 1 else -1
q, k, v = ((torch.rand((bh, 1, s, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
tr = torch.zeros((12 * 1024,), dtype=torch.int64, device="cuda")
for _ in range(2):
    P.attention_fwd(q, k, v, emu=emu)
tr.zero_()
P.attention_fwd(q, k, v, emu=emu, trace=tr)
torch.cuda.synchronize()
t = tr.cpu().view(12, 1024)


def evs(w):
    out = []
    for x in t[w].tolist():
        if x == 0:
            break
        out.append((x >> 8, x & 0xFF))
    return out


mma, w0, w4 = sorted(evs(9) + evs(10)), evs(0), evs(4)
t0 = mma[0][0]
names = {1: "S0", 2: "PV0", 3: "S1", 4: "PV1", 20: "V", 21: "S0i", 22: "PV0i", 23: "S1i", 24: "PV1i"}
sm = {10: "sfull", 15: "ld1", 16: "mx1", 11: "ld", 12: "sfree", 13: "pvok", 14: "P"}
# group MMA events into steps at each S0 issue
steps, cur = [], None
for ts, c in mma:
    if c == 1:
        cur = {"S0": ts}
        steps.append(cur)
    elif cur is not None:
        cur.setdefault(names[c], ts)
w0s = [e for e in w0]
w4s = [e for e in w4]
print("step | S0  PV0  S1  PV1 (abs, rel to S0) | period")
prev = None
for i, st in enumerate(steps[8:40]):
    base = st["S0"]
    rel = " ".join(f"{n}:{st.get(n, 0) - base:6d}" for n in ("PV0", "S1", "PV1"))
    print(f"{i + 8:3d} | S0@{base - t0:9d} {rel} | {base - prev if prev else 0}")
    prev = base
print("\nsoftmax WG0 warp0 (per step: sfull, ld, pvok, P) relative to previous P")
for lst, nm in ((w0s, "WG0"), (w4s, "WG1")):
    seq, out = [], []
    for ts, c in lst:
        seq.append((ts, c))
    # split into steps by code 10
    stp, cur = [], []
    for ts, c in seq:
        if c == 10 and cur:
            stp.append(cur)
            cur = []
        cur.append((ts, c))
    for i, st in enumerate(stp[8:24]):
        b = st[0][0]
        print(nm, i + 8, "  ".join(f"{sm[c]}:{ts - b:5d}" for ts, c in st), f" @{b - t0}")

print("\nper-warp P publish time (rel. to warp 0 / warp 4 of the same WG), steps 8..15")
allw = [evs(w) for w in range(8)]


def p_times(lst):
    return [ts for ts, c in lst if c == 14]


def ld_times(lst):
    return [ts for ts, c in lst if c == 11]


for wg in (0, 1):
    base = p_times(allw[4 * wg])
    bl = ld_times(allw[4 * wg])
    for i in range(8, 16):
        print(f"WG{wg} step {i}: P " + " ".join(f"{p_times(allw[4 * wg + q])[i] - base[i]:6d}" for q in range(4))
              + "   ld " + " ".join(f"{ld_times(allw[4 * wg + q])[i] - bl[i]:6d}" for q in range(4)))

print("\nMMA warp raw events of steps 10..12 (code: 1 S0 ok-to-issue, 21 S0 issued, 20 V ready,"
      " 2 PV0 ok, 22 PV0 issued, 3 S1 ok, 23 S1 issued, 4 PV1 ok, 24 PV1 issued)")
st = [i for i, (ts, c) in enumerate(mma) if c == 1]
a, b = st[10], st[13]
base = mma[a][0]
print("  ".join(f"{c}:{ts - base}" for ts, c in mma[a:b]))

print("\nsoftmax events in the same window (rel. to the MMA window base): code 10 sfull, 11 ld(S free), 13 pv-ok, 14 P")
for w in range(8):
    ev = [(ts - base, c) for ts, c in allw[w] if base - 4000 <= ts <= mma[b][0]]
    print(f"warp {w}: " + "  ".join(f"{c}:{ts}" for ts, c in ev))
