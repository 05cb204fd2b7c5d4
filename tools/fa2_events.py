"""Timeline of cluster 0 of the 2-CTA attention kernel (debug aid; run with
--build, which compiles an event build (-DMIMW_FA_EVENTS) into /tmp).
Per KV step: when the leader issued S(j) / PV(j), and when CTA 0 / CTA 1
softmax warp 0 saw S, released it, had the row max, finished the
exponentials, had PV(j-2) done and published P (cycles)."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "--build" in sys.argv:
    dst = "/tmp/mimw_fa_events"
    shutil.rmtree(dst, ignore_errors=True)
    shutil.copytree(os.path.join(ROOT, "paper_2605_10905_b200"), os.path.join(dst, "paper_2605_10905_b200"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(dst, "include"))
    env = {**os.environ, "MIMW_NVCC_EXTRA": "-DMIMW_FA_EVENTS"}
    subprocess.run([sys.executable, "-c", "import paper_2605_10905_b200.build as b; b.build(force=True)"],
                   cwd=dst, env=env, check=True)
    env = {**os.environ, "MIMW_B200_LIB": os.path.join(dst, "paper_2605_10905_b200", "libmimw_b200.so")}
    sys.exit(subprocess.run([sys.executable, __file__] + [a for a in sys.argv[1:] if a != "--build"],
                            env=env).returncode)

import torch  # noqa: E402
sys.path.insert(0, ROOT)
import paper_2605_10905_b200 as P  # noqa: E402

bh, s = 128, 8192
emu = int(sys.argv[1]) if len(sys.argv) > 1 else -1
q, k, v = ((torch.rand((bh, 1, s, 128), device="cuda") * 2 - 1).bfloat16() for _ in range(3))
tr = torch.zeros((2 * 12 * 1024,), dtype=torch.int64, device="cuda")
for _ in range(2):
    P.attention_fwd(q, k, v, emu=emu)
tr.zero_()
P.attention_fwd(q, k, v, emu=emu, trace=tr)
torch.cuda.synchronize()
t = tr.cpu().view(2, 12, 1024)


def evs(r, w):
    out = []
    for x in t[r, w].tolist():
        if x == 0:
            break
        out.append((x >> 8, x & 0xFF))
    return out


S = [e for e in evs(0, 9)]
PV = [e for e in evs(0, 10)]
t0 = S[0][0]
s_iss = [ts for ts, c in S if c == 3]
s_req = [ts for ts, c in S if c == 1]
s_got = [ts for ts, c in S if c == 2]
pv_req = [ts for ts, c in PV if c == 4]
pv_got = [ts for ts, c in PV if c == 5]
pv_iss = [ts for ts, c in PV if c == 6]
print("step | S: want_free got_free issued | PV: wait got issued | period(S issued)")
for j in range(4, min(40, len(s_iss), len(pv_iss))):
    print(f"{j:3d} | {s_req[j] - t0:8d} {s_got[j] - t0:8d} {s_iss[j] - t0:8d} | {pv_req[j] - t0:8d} "
          f"{pv_got[j] - t0:8d} {pv_iss[j] - t0:8d} | {s_iss[j] - s_iss[j - 1]}")
names = {10: "sfull", 16: "ld", 11: "sfree", 18: "exps", 19: "hand", 12: "pub", 13: "pack", 14: "pvok", 17: "st", 15: "P"}
for r in (0, 1):
    ev = evs(r, 0)
    steps, cur = [], []
    for ts, c in ev:
        if c == 10 and cur:
            steps.append(cur)
            cur = []
        cur.append((ts, c))
    print(f"\nCTA {r} softmax warp 0, relative to S seen (abs = cycles since first S issue)")
    for j, st in enumerate(steps[4:24]):
        b = st[0][0]
        print(f"{j + 4:3d} @{b - t0:8d} " + "  ".join(f"{names[c]}:{ts - b:5d}" for ts, c in st))
prod = evs(0, 8)
print("\nproducer CTA 0: slot-free times (K=30, V=31) for the first 24 loads")
print(" ".join(f"{c - 30}:{ts - t0}" for ts, c in prod[:24]))
