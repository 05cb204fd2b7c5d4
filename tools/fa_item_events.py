"""Item-boundary timeline of CTA 0 of the attention kernel (debug aid; build
with MIMW_NVCC_EXTRA=-DMIMW_FA_EVENTS).  For each work item: when the S
issuer issued its first/last S, when each softmax warpgroup finished its last
step, ran the epilogue (O / l to HBM), and when the producer saw Q released
and issued the next item's Q loads.  Cycles relative to the first S."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10905_b200 as P  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 2048
bh = max(1, 128 * (8192 // s) ** 2 // 64)
q, k, v = ((torch.rand((bh, 1, s, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
tr = torch.zeros((12 * 1024,), dtype=torch.int64, device="cuda")
for _ in range(2):
    P.attention_fwd(q, k, v, causal=False)
tr.zero_()
P.attention_fwd(q, k, v, causal=False, trace=tr)
torch.cuda.synchronize()
t = tr.cpu().view(12, 1024)


def evs(w):
    out = []
    for x in t[w].tolist():
        if x == 0:
            break
        out.append((x >> 8, x & 0xFF))
    return out


t0 = min(ts for w in (9, 10) for ts, _ in evs(w))
names = {1: "S0", 3: "S1", 2: "PV0", 4: "PV1", 10: "sfull", 11: "ld", 14: "P", 30: "epi0", 31: "epi1",
         40: "Qrel0", 41: "Qrel1", 32: "item", 33: "publish"}
rows = []
for w, who in ((9, "mma-S"), (10, "mma-PV"), (0, "wg0"), (4, "wg1"), (8, "prod")):
    for ts, c in evs(w):
        if c in (30, 31, 32, 33, 40, 41) or (w in (9, 10) and c in (1, 2, 3, 4)) or (w in (0, 4) and c in (10, 11, 14)):
            rows.append((ts - t0, who, names.get(c, str(c))))
rows.sort()
# print around the first few item boundaries (epilogue events)
epis = [r for r in rows if r[2] == "epi0" and r[1] == "wg0"]
for e in epis[:4]:
    print(f"---- item boundary near {e[0]} ----")
    for r in rows:
        if e[0] - 6000 <= r[0] <= e[0] + 9000 and r[2] not in ("PV0", "PV1") or (
                e[0] - 3000 <= r[0] <= e[0] + 6000):
            print(f"{r[0]:9d} {r[1]:7s} {r[2]}")

# steady-state step period (S0 -> S0 within an item) vs periods spanning an item boundary
s0 = [ts for ts, c in evs(9) if c == 1]
ep = sorted(ts for ts, c in evs(0) if c == 30)
per = [b - a for a, b in zip(s0, s0[1:])]
inner = [p for p, a in zip(per, s0) if not any(a < e < a + p for e in ep)]
cross = [p for p, a in zip(per, s0) if any(a < e < a + p for e in ep)]
if inner:
    inner.sort()
    print(f"S={s}: S0 period median {inner[len(inner) // 2]} cycles over {len(inner)} in-item steps; "
          f"boundary periods {sorted(cross)[:6]}")

if "--raw" in sys.argv:
    b0 = [ts for ts, c in evs(0) if c == 30][1]
    print("\nraw events (warp: code@cycle rel. to the 2nd epilogue of warp 0)")
    for w in (0, 4, 8, 9, 10):
        print(f"warp {w}: " + "  ".join(f"{c}@{ts - b0}" for ts, c in evs(w) if -6000 <= ts - b0 <= 8000))
    print("producer all: " + "  ".join(f"{c}@{ts - b0}" for ts, c in evs(8)[:40]))
    print("S-warp S0 issues: " + "  ".join(f"{ts - b0}" for ts, c in evs(9) if c == 1)[:600])
    print("warp0 item/epi: " + "  ".join(f"{c}@{ts - b0}" for ts, c in evs(0) if c in (30, 31, 32))[:600])
