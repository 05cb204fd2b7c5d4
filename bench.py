#!/usr/bin/env python3
"""Benchmark of the B200 hot path (BASELINE.json metric: GEMM/FA-fwd TFLOPS
per B200 and % of dense tensor peak; 1/2/4/8-GPU scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload gemm|attention|all]

Default workload = BASELINE.json configs[1]: persistent warp-specialized bf16
GEMM M=N=K=8192 (2-CTA clusters + TMA multicast) on each GPU.  A "step" is
one launch of the kernel over one 8192^3 problem.  N>1 (torchrun, one rank
per GPU, NCCL): every rank runs its own independent 8192^3 GEMM ("GEMM
batches", weak scaling, no data-path collective); value = total FLOP of all
ranks / max-over-ranks device time.

Timing: W warm-up steps, then exactly K steps bracketed by barrier +
cuda.synchronize, CUDA events on the launching stream, max over ranks.
Inputs A, B are 2 x 128 MiB bf16 > 126 MB L2 (no L2 flush needed; stated in
config).  nvidia-smi clocks are sampled during the timed region.

--impl reference: the reference's own CPU path (oracle/_ref, compiled from
/root/reference/proj/core/src/oracles.cpp, oracle_gemm / oracle_attention)
timed on this host's cores with all threads, each step a bounded row/head
sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GEMM_M = GEMM_N = GEMM_K = 8192
FA_B, FA_H, FA_S, FA_D = 4, 32, 8192, 128
METRIC = "GEMM/FA-fwd TFLOPS per B200 and % of dense tensor peak; 1/2/4/8-GPU scaling"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(bf16=d["bf16_tflops"], bf16_sustained=d.get("bf16_tflops_sustained"),
                    hbm=d["hbm_gbs"], src="measured")
    return dict(bf16=1590.0, bf16_sustained=1400.0, hbm=6650.0, src="fallback")


def traffic(key):
    """DRAM bytes per launch of the kernel from the committed ncu capture
    (profiles/traffic.json, written from `ncu --set full` via tools/profile.sh)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[key]["bytes"]
    except (OSError, KeyError, ValueError):
        return None


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.limit")
    # clocks_event_reasons.active bit mask (nvml): reasons the per-reason columns do not cover
    MASK = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
            0x100: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()
        # nvidia-smi needs a few hundred ms to emit its first sample: wait for
        # it, then keep only the samples taken from here on (the timed region
        # of a ~100-ms workload would otherwise see none)
        t_end = time.time() + 3.0
        while not self.rows and time.time() < t_end:
            time.sleep(0.01)
        self.rows.clear()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(1)
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = {names[i] for r in self.rows if len(r) >= 8
                   for i in range(4) if r[4 + i].lower().startswith("active")}
        for r in self.rows:
            if len(r) >= 8:
                try:
                    bits = int(r[3], 16)
                except ValueError:
                    continue
                reasons |= {v for k, v in self.MASK.items() if bits & k}
        reasons = sorted(reasons)
        # "under load": samples drawing > 40% of the peak power seen (the 50-ms
        # sampler also catches the idle edges around a short timed region)
        pw = [float(r[2]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()
              and r[2].replace(".", "").isdigit()]
        if len(pw) == len(sm) and pw:
            loaded = [s_ for s_, w_ in zip(sm, pw) if w_ > 0.4 * max(pw)]
        else:
            loaded = [s_ for s_ in sm if s_ > 500]
        loaded = loaded or sm
        lim = [float(r[8]) for r in self.rows if len(r) >= 9 and r[8].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm),
                # the 1 kW cap: a clock below max with the draw at the limit is power, not a lock
                "power_w_max": max(pw) if pw else None, "power_limit_w": max(lim) if lim else None}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def backend_for(ws: int) -> str:
    """nccl (one rank per GPU), or gloo when MIMW_BENCH_BACKEND says so or the
    box has fewer GPUs than ranks (ranks then share GPUs: a functional check
    of the multi-rank path, not a scaling measurement)."""
    import torch
    b = os.environ.get("MIMW_BENCH_BACKEND")
    if b:
        return b
    return "nccl" if torch.cuda.device_count() >= ws else "gloo"


def dist_init(n_gpus):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws != n_gpus:
        raise SystemExit(f"bench.py: --gpus {n_gpus} but WORLD_SIZE={ws} ranks were launched")
    if ws > 1:
        import torch.distributed as dist
        backend = backend_for(ws) if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        assert dist.get_world_size() == n_gpus
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, ws, local


def relaunch(n_gpus: int) -> int:
    """`bench.py --gpus N` (N > 1) started as a plain process: re-exec under
    torchrun with one rank per GPU (127.0.0.1 rendezvous), NCCL_DEBUG=INFO so
    the communicator's rank count is visible; returns torchrun's exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def e2e_h2d_bytes(m, n, k):
    """H2D bytes of one mimw_b200_oracle_gemm call (PREC_BF16), following the
    chunking of capi.cu host_gemm_host_staged: row chunks of B (k/8 rows) and A
    (m/8 rows); MIMW_HOST_STAGE 0 = all f32, 1 = all bf16, 2 = B's odd chunks
    and all of A f32, 3 (default) = odd chunks of both f32, the rest bf16."""
    mode = int(os.environ.get("MIMW_HOST_STAGE", "3"))
    r8 = lambda x, q: (x + q - 1) // q * q  # noqa: E731
    kp, np_ = r8(k, 8), r8(n, 8)
    if mode == 0:
        return 4 * (m * k + k * n)
    bchunk = max(64, r8((k + 7) // 8, 8))
    achunk = max(512, r8((m + 7) // 8, 256))
    total = 0
    for i, r0 in enumerate(range(0, k, bchunk)):
        rows = min(bchunk, k - r0)
        total += 4 * rows * n if (mode != 1 and i % 2 == 1) else 2 * rows * np_
    for i, r0 in enumerate(range(0, m, achunk)):
        rows = min(achunk, m - r0)
        f32 = mode == 2 or (mode == 3 and i % 2 == 1)
        total += 4 * rows * k if f32 else 2 * rows * kp
    return total


COOLDOWN_S = 2.0


def cooldown(ws):
    """Idle COOLDOWN_S seconds (all ranks) between the line's workloads."""
    import torch
    torch.cuda.synchronize()
    time.sleep(COOLDOWN_S)
    barrier(ws)


def timed(step, steps, warmup, ws, stream):
    """W warm-up steps, then K steps between barrier+synchronize, CUDA events
    on the launching stream; returns max-over-ranks seconds for the K steps."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    return max_over_ranks(e0.elapsed_time(e1) / 1e3, ws)


def reassembly_ms(fn, ws, reps=5):
    """Device time of one output reassembly (NCCL all-gather over NVLink),
    max over ranks; reported next to the compute-only value."""
    import torch
    fn()
    torch.cuda.synchronize()
    barrier(ws)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / reps, ws)
    import torch.distributed as dist
    be = dist.get_backend()
    op = "ncclAllGather" if be == "nccl" else f"{be} all-gather"
    return {"op": f"{op} (torch.distributed all_gather_into_tensor / all_gather)", "backend": be,
            "ms": round(ms, 4)}


# ---------------------------------------------------------------------------
# CPU reference path (oracle/_ref = the unmodified reference oracles)
# ---------------------------------------------------------------------------
def cpu_gemm_sample(seconds_target: float = 12.0, single: bool = True):
    """Time oracle_gemm (oracles.cpp:14-26) on a row sample of the 8192^3
    workload with all host threads (one row block each), plus the as-shipped
    single-thread rate on a 2-row sample; returns a cpu_baseline dict."""
    import oracle
    R = oracle.REF
    kind = "reference"
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(7)
    b = oracle.round_bf16(rng.uniform(-1, 1, (GEMM_K, GEMM_N)).astype(np.float32))
    rows = threads
    a = oracle.round_bf16(rng.uniform(-1, 1, (rows, GEMM_K)).astype(np.float32))

    def run(nr, thr):
        c = np.empty((nr, GEMM_N), np.float32)
        t0 = time.perf_counter()
        if R is not None:
            R.ref_oracle_gemm_mt(a[:nr].copy(), b, c, nr, GEMM_N, GEMM_K, thr)
        else:
            oracle.oracle_gemm(a[:nr], b)
        return time.perf_counter() - t0

    if R is None:
        kind, threads = "port", 1
        rows = 1
    dt = run(rows, threads)
    if R is not None and dt < seconds_target / 3:
        per = int(min(16, max(1, round(seconds_target / max(dt, 1e-3)))))
        rows = threads * per
        a = oracle.round_bf16(rng.uniform(-1, 1, (rows, GEMM_K)).astype(np.float32))
        dt = run(rows, threads)
    flops = 2.0 * rows * GEMM_N * GEMM_K
    one = None
    if R is not None and threads > 1 and single:
        dt1 = run(2, 1)
        one = 2.0 * 2 * GEMM_N * GEMM_K / dt1 / 1e12
    return {"value": flops / dt / 1e12, "unit": "TFLOPS", "cores": threads, "kind": kind,
            "sample": f"{rows} of {GEMM_M} rows of the 8192^3 GEMM ({threads} threads, one row block each), "
                      f"{dt:.1f} s; whole-GEMM time extrapolated x{GEMM_M / rows:.1f} (rows are independent, "
                      "oracles.cpp:17-23)",
            "extrapolation_factor": round(GEMM_M / rows, 2),
            "single_thread_value": one,
            "single_thread_sample": "2 rows, 1 thread (the reference as shipped is single-threaded)"}


def cpu_attention_sample(seq: int = 4096):
    """Time oracle_attention (oracles.cpp:119-145) on `threads` causal heads of
    [seq, 128] with all host threads (one head each); returns a cpu_baseline
    dict in TFLOPS (causal FA FLOP convention)."""
    import oracle
    R = oracle.REF
    threads = os.cpu_count() or 1
    heads = threads
    s, d = seq, FA_D
    rng = np.random.default_rng(31)
    q, k, v = (oracle.round_bf16(rng.uniform(-1, 1, (heads, s, d)).astype(np.float32))
               for _ in range(3))
    o = np.empty_like(q)
    t0 = time.perf_counter()
    if R is not None:
        R.ref_oracle_attention_heads_mt(q, k, v, o, heads, s, d, s, 1 / np.sqrt(d), threads)
        kind = "reference"
    else:
        oracle.oracle_attention(q[0], k[0], v[0], s, 1 / np.sqrt(d))
        heads, threads, kind = 1, 1, "port"
    dt = time.perf_counter() - t0
    flops = 4.0 * heads * d * s * (s + 1) / 2
    return {"value": flops / dt / 1e12, "unit": "TFLOPS", "cores": threads, "kind": kind,
            "sample": f"{heads} causal heads S={s} D={d} ({threads} threads, one head each), {dt:.1f} s; "
                      f"configs[3] has {FA_B * FA_H} heads of S={FA_S} (cost ~S^2: one S={FA_S} head = "
                      f"{(FA_S / s) ** 2:.0f}x a sampled head)"}


# ---------------------------------------------------------------------------
# our GEMM
# ---------------------------------------------------------------------------
def bench_gemm(args, rank, ws, local):
    import torch
    import paper_2605_10905_b200 as P
    P.lib()
    pk = peaks()
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    a = (torch.rand((GEMM_M, GEMM_K), device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand((GEMM_K, GEMM_N), device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    c = torch.empty((GEMM_M, GEMM_N), device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    L = P.lib()

    def step():
        P._check(L.mimw_b200_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), GEMM_M, GEMM_N,
                                       GEMM_K, GEMM_K, GEMM_N, GEMM_N, P.B_KN, P.BF16, sptr))

    clk = Clocks(local)
    clk.start()
    secs = timed(step, args.steps, args.warmup, ws, stream)
    clocks = clk.stop()
    flop = 2.0 * GEMM_M * GEMM_N * GEMM_K
    per_launch = secs / args.steps
    value = ws * flop * args.steps / secs / 1e12
    achieved = flop / per_launch / 1e12

    # same-box cuBLAS (torch.mm on the same operands) for context
    cublas = None
    try:
        csecs = timed(lambda: torch.mm(a, b, out=c), args.steps, args.warmup, ws, stream)
        cublas = round(flop * args.steps / csecs / 1e12, 2)
    except Exception as e:  # noqa: BLE001
        cublas = f"unavailable: {type(e).__name__}"
    # the design alternatives on the same operands, same box: the 256x256 pair
    # tile, and clusters of two pairs sharing each B k-block by TMA multicast
    # (north_star's "2-CTA cluster mode with TMA multicast")
    alts = {}
    for name, kw in (("tile_256x256", dict(tile_n=256)), ("tma_multicast_two_pairs", dict(cta_group=4))):
        try:
            asecs = timed(lambda kw=kw: P.gemm(a, b, out=c, **kw), args.steps, args.warmup, ws, stream)
            alts[name] = round(flop * args.steps / asecs / 1e12, 2)
        except Exception as e:  # noqa: BLE001
            alts[name] = f"unavailable: {type(e).__name__}"

    # end to end through the reference-facing C-ABI with HOST f32 buffers
    # (mimw_b200_oracle_gemm: H2D of A, B, bf16 staging, GEMM, D2H of C), with
    # pageable buffers as the reference's Tile (std::vector, sim.hpp:13-26)
    # and with pinned ones
    e2e = None
    if not args.no_e2e:
        import ctypes
        fp = P._fp
        ha_pg = a.float().cpu().numpy()
        hb_pg = b.float().cpu().numpy()
        hc_pg = np.empty((GEMM_M, GEMM_N), np.float32)
        hc_pg.fill(0)  # touch the pages once (a caller's Tile is resident)
        ha = torch.from_numpy(ha_pg).pin_memory()
        hb = torch.from_numpy(hb_pg).pin_memory()
        hc = torch.empty((GEMM_M, GEMM_N), dtype=torch.float32).pin_memory()

        def e2e_time(pa, pb, pc):
            def e2e_step():
                P._check(L.mimw_b200_oracle_gemm(ctypes.cast(pa, fp), ctypes.cast(pb, fp), ctypes.cast(pc, fp),
                                                 GEMM_M, GEMM_N, GEMM_K, P.PREC_BF16))
            for _ in range(2):
                e2e_step()
            barrier(ws)
            n_e2e = max(3, min(10, args.steps // 4))
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                e2e_step()
            return max_over_ranks((time.perf_counter() - t0) / n_e2e, ws)

        dt_pg = e2e_time(ha_pg.ctypes.data, hb_pg.ctypes.data, hc_pg.ctypes.data)
        dt_pin = e2e_time(ha.data_ptr(), hb.data_ptr(), hc.data_ptr())
        e2e = {"value": round(ws * flop / dt_pg / 1e12, 2), "unit": "TFLOPS",
               "h2d_bytes_per_step": e2e_h2d_bytes(GEMM_M, GEMM_N, GEMM_K),
               "d2h_bytes_per_step": 4 * GEMM_M * GEMM_N,
               "api": "mimw_b200_oracle_gemm (host f32 Tiles, include/mimw_b200.h)",
               "ms_per_step": round(dt_pg * 1e3, 3),
               "host_buffers": "pageable (numpy, as the reference's std::vector Tile)",
               "pinned": {"value": round(ws * flop / dt_pin / 1e12, 2), "ms_per_step": round(dt_pin * 1e3, 3)},
               "pageable": {"value": round(ws * flop / dt_pg / 1e12, 2), "ms_per_step": round(dt_pg * 1e3, 3)}}

    res = {
        "metric": METRIC, "value": round(value, 2), "unit": "TFLOPS", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic U[-1,1] bf16 (random init, no dataset)",
        "config": {"workload": "configs[1]: warp-specialized bf16 GEMM M=N=K=8192 (tiles by cluster launch control), "
                               "2-CTA clusters (cta_group::2), fp32 accumulate in TMEM, bf16 out",
                   "M": GEMM_M, "N": GEMM_N, "K": GEMM_K,
                   "tile": "256x512x64 per CTA pair (gemm_wide.cuh), 4-stage ring, register-drained epilogue",
                   "parallelism": f"{ws} independent GEMM batches (one per GPU)",
                   "l2": "inputs 2 x 128 MiB > 126 MB L2 (no flush)"},
        "roofline": {"bound": "tensor", "achieved": round(achieved, 2),
                     "peak": pk["bf16"], "unit": "TFLOP/s", "frac": round(achieved / pk["bf16"], 4),
                     "peak_source": f"{pk['src']} bf16 burst (MEASURED_PEAKS.json)",
                     "frac_of_spec_2250": round(achieved / 2250.0, 4),
                     "traffic": traffic("gemm_bf16_8192"),
                     "cublas_tflops_same_box": cublas,
                     "alternatives_tflops_same_box": alts,
                     "algorithmic_bytes_min": 2.0 * (GEMM_M * GEMM_K + GEMM_K * GEMM_N + GEMM_M * GEMM_N),
                     "algorithmic_flop_per_launch": flop},
        "e2e": e2e,
        "gpu_launches": args.steps,
        "clocks": clocks,
    }
    return res


def bench_attention(args, rank, ws, local):
    """configs[3]: causal FA forward bf16 B=4 H=32 S=8192 D=128, batch x head
    sharded over the ranks (strong scaling: each rank runs B*H/N heads).
    Timed for the full --steps; e2e through the host-f32 reference-signature
    entries; the reference oracle_attention timed on the host cores; cuDNN
    SDPA timed on the same inputs for context."""
    import ctypes
    import torch
    import paper_2605_10905_b200 as P
    L = P.lib()
    pk = peaks()
    dev = torch.device("cuda", local)
    from paper_2605_10905_b200 import shard
    bh = FA_B * FA_H
    ranges = shard.head_shards(bh, ws)
    my = ranges[rank][1] - ranges[rank][0]
    g = torch.Generator(device=dev).manual_seed(31 + rank)
    q, k, v = ((torch.rand((my, 1, FA_S, FA_D), device=dev, generator=g) * 2 - 1)
               .to(torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty((my, 1, FA_S), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    scale = FA_D ** -0.5

    def step():
        P._check(L.mimw_b200_attention_fwd_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                              lse.data_ptr(), my, 1, FA_S, FA_S, scale, args.fa_emu,
                                              0, None, 1, sptr))

    steps = args.steps
    clk = Clocks(local)
    clk.start()
    secs = timed(step, steps, args.warmup, ws, stream)
    clocks = clk.stop()
    flop_total = 4.0 * bh * FA_D * FA_S * FA_S / 2  # FA causal convention
    flop_mine = flop_total / ws
    value = flop_total * steps / secs / 1e12
    achieved = flop_mine / (secs / steps) / 1e12
    reasm = None
    if ws > 1:  # all-gather of O and LSE, reported beside (not inside) the compute number
        reasm = reassembly_ms(lambda: (shard.all_gather_rows(o, ranges),
                                       shard.all_gather_rows(lse, ranges)), ws)
        reasm["bytes_gathered"] = bh * FA_S * (FA_D * 2 + 4)
    # cuDNN SDPA (torch) on the same inputs, same box, for context
    cudnn = None
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            f = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)  # noqa: E731
            cs = timed(f, steps, args.warmup, ws, stream)
        cudnn = round(flop_total * steps / cs / 1e12, 2)
    except Exception as e:  # noqa: BLE001
        cudnn = f"unavailable: {type(e).__name__}"
    # end to end through the host-f32 reference-signature entries, pageable
    # numpy buffers (the reference's Tile): (a) the batched entry, all of this
    # rank's heads in one call; (b) the per-head oracle_attention signature
    # called once per head
    e2e = None
    if not args.no_e2e:
        hq, hk, hv = (t.reshape(my, FA_S, FA_D).float().cpu().numpy() for t in (q, k, v))
        ho = np.zeros((my, FA_S, FA_D), np.float32)
        hl = np.zeros((my, FA_S), np.float32)
        fp = P._fp
        cp = lambda x: ctypes.cast(x.ctypes.data, fp)  # noqa: E731

        def batched():
            P._check(L.mimw_b200_oracle_attention_heads(cp(hq), cp(hk), cp(hv), cp(ho), cp(hl), my, FA_S,
                                                        FA_D, FA_S, scale, P.PREC_BF16))

        def per_head():
            for h in range(my):
                P._check(L.mimw_b200_oracle_attention_ex(cp(hq[h]), cp(hk[h]), cp(hv[h]), cp(ho[h]), cp(hl[h]),
                                                         FA_S, FA_D, FA_S, scale, P.PREC_BF16))

        def wall(fn, n):
            fn()
            barrier(ws)
            t0 = time.perf_counter()
            for _ in range(n):
                fn()
            return max_over_ranks((time.perf_counter() - t0) / n, ws)

        dt = wall(batched, max(3, min(10, args.steps // 4)))
        dt_ph = wall(per_head, 2)
        elems = my * FA_S * FA_D
        e2e = {"value": round(flop_total / dt / 1e12, 2), "unit": "TFLOPS",
               "h2d_bytes_per_step": 3 * 2 * my * FA_S * 128,
               "d2h_bytes_per_step": 2 * my * FA_S * 128 + 4 * my * FA_S,
               "ms_per_step": round(dt * 1e3, 3),
               "api": "mimw_b200_oracle_attention_heads (host f32 [H,S,D], pageable numpy; f32<->bf16 on "
                      "host threads, PCIe at 2 B/element)",
               "host_f32_bytes_per_step": 4 * 4 * elems,
               "per_head_reference_signature": {
                   "value": round(flop_total / dt_ph / 1e12, 2), "ms_per_step": round(dt_ph * 1e3, 3),
                   "api": f"mimw_b200_oracle_attention_ex called {my} times (one [S,D] head per call, "
                          "the reference's oracle_attention signature)"}}
    res = {"metric": METRIC, "value": round(value, 2), "unit": "TFLOPS", "n_gpus": ws,
           "steps": steps, "warmup": args.warmup, "ms_per_step": round(secs / steps * 1e3, 4),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
           "reassembly": reasm,
           "data": "synthetic U[-1,1] bf16",
           "config": {"workload": "configs[3]: causal flash-attention forward bf16 B=4 H=32 "
                                  "S=8192 D=128, batch x head sharded",
                      "B": FA_B, "H": FA_H, "S": FA_S, "D": FA_D,
                      "parallelism": f"{my} of {bh} heads per GPU",
                      "l2": "Q,K,V 3 x 256 MiB > 126 MB L2 (no flush)"},
           "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": pk["bf16"],
                        "unit": "TFLOP/s", "frac": round(achieved / pk["bf16"], 4),
                        "frac_of_spec_2250": round(achieved / 2250.0, 4),
                        "peak_source": f"{pk['src']} bf16 burst (MEASURED_PEAKS.json)",
                        "traffic": traffic("attention_fwd_b4h32s8192") if ws == 1 else None,
                        "algorithmic_flop_per_launch": flop_mine,
                        "cudnn_sdpa_tflops_same_box": cudnn},
           "e2e": e2e, "gpu_launches": steps, "clocks": clocks}
    return res


def bench_mxfp8(args, rank, ws, local):
    """configs[2]: FP8 (e4m3) block-scaled GEMM M=N=K=8192 (MXFP8, UE8M0 per
    1x32 along K), one independent GEMM per GPU (weak scaling)."""
    import torch
    import paper_2605_10905_b200 as P
    L = P.lib()
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(3 + rank)
    m = n = k = GEMM_M
    qa = torch.randint(0, 256, (m, k), device=dev, dtype=torch.uint8, generator=g)
    qb = torch.randint(0, 256, (n, k), device=dev, dtype=torch.uint8, generator=g)
    qa[(qa & 0x7F) == 0x7F] = 0x38
    qb[(qb & 0x7F) == 0x7F] = 0x38
    sfa = torch.randint(120, 134, (m, k // 32), device=dev, dtype=torch.uint8, generator=g)
    sfb = torch.randint(120, 134, (n, k // 32), device=dev, dtype=torch.uint8, generator=g)
    c = torch.empty((m, n), device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def step():
        P._check(L.mimw_b200_gemm_mxfp8(qa.data_ptr(), sfa.data_ptr(), qb.data_ptr(), sfb.data_ptr(),
                                        c.data_ptr(), m, n, k, sptr))

    steps = args.steps
    clk = Clocks(local)
    clk.start()
    secs = timed(step, steps, args.warmup, ws, stream)
    clocks = clk.stop()
    flop = 2.0 * m * n * k
    achieved = flop / (secs / steps) / 1e12
    # cuBLAS FP8 (torch._scaled_mm, per-tensor scales) on the same box as a reference point
    ref = None
    try:
        a8 = qa.view(torch.float8_e4m3fn)
        b8 = qb.view(torch.float8_e4m3fn)
        one = torch.ones((), device=dev)
        f = lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        rs = timed(f, 10, 3, 1, stream)
        ref = round(flop * 10 / rs / 1e12, 1)
    except Exception as e:  # noqa: BLE001
        ref = f"unavailable: {type(e).__name__}"
    # cuBLAS MXFP8 (the same 1x32 UE8M0 block scaling; scales handed over already
    # in cuBLAS's swizzled layout, so its time excludes any scale reordering)
    ref_mx = None
    try:
        from torch.nn.functional import ScalingType, SwizzleType, scaled_mm
        sa8 = sfa.view(torch.float8_e8m0fnu)
        sb8 = sfb.view(torch.float8_e8m0fnu)
        fm = lambda: scaled_mm(a8, b8.t(), sa8, ScalingType.BlockWise1x32, sb8, ScalingType.BlockWise1x32,
                               swizzle_a=SwizzleType.SWIZZLE_32_4_4, swizzle_b=SwizzleType.SWIZZLE_32_4_4,
                               output_dtype=torch.bfloat16)
        rs = timed(fm, 10, 3, 1, stream)
        ref_mx = round(flop * 10 / rs / 1e12, 1)
    except Exception as e:  # noqa: BLE001
        ref_mx = f"unavailable: {type(e).__name__}"
    return {"value": round(ws * flop * steps / secs / 1e12, 2), "unit": "TFLOPS",
            "ms_per_step": round(secs / steps * 1e3, 4), "scaling": "weak",
            "config": {"workload": "configs[2]: MXFP8 e4m3 block-scaled GEMM M=N=K=8192 "
                                   "(UE8M0 per 1x32 along K), bf16 out, 2-CTA 256x224x128 tiles (cta_group::2); "
                                   "step includes the scale-factor atom reorder pre-pass"},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": 4500.0,
                         "unit": "TFLOP/s", "frac": round(achieved / 4500.0, 4),
                         "peak_source": "spec dense FP8 (no measured FP8 peak in MEASURED_PEAKS.json)",
                         "cublas_fp8_scaled_mm_tflops_same_box": ref,
                         "cublas_mxfp8_scaled_mm_tflops_same_box": ref_mx,
                         "traffic": traffic("mxfp8_8192")},
            "clocks": clocks}


MOE_E, MOE_K, MOE_N, MOE_TOKENS, MOE_TOPK = 64, 4096, 14336, 16384, 2


def moe_counts(seed=5):
    """configs[4] routing: Dirichlet(1) expert probabilities, multinomial
    assignment of tokens * top_k rows."""
    rng = np.random.default_rng(seed)
    p = rng.dirichlet(np.ones(MOE_E))
    return rng.multinomial(MOE_TOKENS * MOE_TOPK, p)


def bench_moe(args, rank, ws, local):
    """configs[4]: grouped MoE GEMM, 64 experts x [4096 x 14336] bf16, ragged
    Dirichlet token counts, sharded by expert (rank r owns experts
    [r*64/N, (r+1)*64/N)); strong scaling (total work fixed)."""
    import torch
    import paper_2605_10905_b200 as P
    L = P.lib()
    pk = peaks()
    dev = torch.device("cuda", local)
    from paper_2605_10905_b200 import shard
    counts = moe_counts()
    parts = shard.expert_shards(counts, ws)
    e0, e1 = parts[rank]
    per = e1 - e0
    mine = counts[e0:e1]
    offs = np.concatenate([[0], np.cumsum(mine)]).astype(np.int64)
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    w = torch.empty((max(1, per), MOE_K, MOE_N), device=dev, dtype=torch.bfloat16)
    for e in range(per):  # chunked init keeps the fp32 temporaries small
        w[e] = (torch.rand((MOE_K, MOE_N), device=dev, generator=g) * 2 - 1).bfloat16()
    x = (torch.rand((max(1, int(offs[-1])), MOE_K), device=dev, generator=g) * 2 - 1).bfloat16()
    y = torch.empty((max(1, int(offs[-1])), MOE_N), device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    offs_c = np.ascontiguousarray(offs)

    def step():
        P._check(L.mimw_b200_grouped_gemm_bf16(x.data_ptr(), offs_c.ctypes.data, w.data_ptr(),
                                               y.data_ptr(), per, MOE_N, MOE_K, P.B_KN, sptr))

    steps = max(3, args.steps // 5) if args.workload != "moe" else args.steps
    clk = Clocks(local)
    clk.start()
    secs = timed(step, steps, args.warmup, ws, stream)
    clocks = clk.stop()
    rows_total = int(counts.sum())
    flop_total = 2.0 * rows_total * MOE_K * MOE_N
    flop_mine = 2.0 * int(offs[-1]) * MOE_K * MOE_N
    per_launch = secs / steps
    achieved = flop_mine / per_launch / 1e12
    bytes_mine = 2.0 * (per * MOE_K * MOE_N + int(offs[-1]) * (MOE_K + MOE_N))
    # same-box library reference: torch._grouped_mm (CUTLASS grouped GEMM in
    # PyTorch) on the same operands and steps, for context only
    lib_ref = None
    try:
        offs_dev = torch.from_numpy(offs[1:].astype(np.int32)).to(dev)
        lsecs = timed(lambda: torch._grouped_mm(x[:int(offs[-1])], w[:per], offs=offs_dev), steps, args.warmup,
                      ws, stream)
        lib_ref = round(flop_mine * steps / lsecs / 1e12, 2)
    except Exception as e:  # noqa: BLE001
        lib_ref = f"unavailable: {type(e).__name__}"
    reasm = None
    if ws > 1:
        full_offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        row_ranges = [shard.group_rows(full_offs, r) for r in parts]
        yl = y[:int(offs[-1])]
        reasm = reassembly_ms(lambda: shard.all_gather_rows(yl, row_ranges), ws)
        reasm["bytes_gathered"] = int(counts.sum()) * MOE_N * 2
    return {"reassembly": reasm, "metric": METRIC, "value": round(flop_total * steps / secs / 1e12, 2), "unit": "TFLOPS",
            "n_gpus": ws, "steps": steps, "warmup": args.warmup,
            "ms_per_step": round(per_launch * 1e3, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic U[-1,1] bf16; Dirichlet(1)/multinomial routing, seed 5",
            "config": {"workload": "configs[4]: grouped MoE GEMM, 64 experts x 4096x14336 bf16, "
                                   "ragged token counts, sharded by expert",
                       "experts": MOE_E, "K": MOE_K, "N": MOE_N,
                       "rows": rows_total, "rows_min_max": [int(counts.min()), int(counts.max())],
                       "parallelism": f"experts [{e0},{e1}) of {MOE_E} on rank {rank} "
                                      "(contiguous min-max tile partition)",
                       "l2": "weights 7.5 GB > 126 MB L2 (no flush)"},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": pk["bf16"],
                         "unit": "TFLOP/s", "frac": round(achieved / pk["bf16"], 4),
                         "peak_source": f"{pk['src']} bf16 burst (MEASURED_PEAKS.json)",
                         "hbm_gbs_min_bytes": round(bytes_mine / per_launch / 1e9, 1),
                         "hbm_peak_gbs": pk["hbm"],
                         "traffic": traffic("grouped_moe") if ws == 1 else None,
                         "algorithmic_flop_per_launch": flop_mine,
                         "torch_grouped_mm_tflops_same_box": lib_ref},
            "gpu_launches": steps, "clocks": clocks}


def bench_layernorm(args, rank, ws, local):
    """cluster LayerNorm, PAPER.md:736 LN6 (1152 x 65536
    f32), rows split across ranks; HBM-bound: 4 B read + 4 B written per element."""
    import torch
    import paper_2605_10905_b200 as P
    L = P.lib()
    pk = peaks()
    dev = torch.device("cuda", local)
    rows_total, n = 1152, 65536
    from paper_2605_10905_b200 import shard
    r0, r1 = shard.split_even(rows_total, ws)[rank]
    rows = r1 - r0
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    x = torch.randn((max(1, rows), n), device=dev, generator=g)
    w = torch.randn(n, device=dev, generator=g)
    b = torch.randn(n, device=dev, generator=g)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def step():
        P._check(L.mimw_b200_layernorm(x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr(), None,
                                       None, rows, n, 1e-5, sptr))

    steps = max(500, args.steps)  # ~55 ms: long enough for the 50-ms clock sampler
    clk = Clocks(local)
    clk.start()
    secs = timed(step, steps, args.warmup, ws, stream)
    clocks = clk.stop()
    per = secs / steps
    gbs = 8.0 * rows * n / per / 1e9
    return {"value": round(8.0 * rows_total * n * steps / secs / 1e9, 1), "unit": "GB/s",
            "ms_per_step": round(per * 1e3, 4), "scaling": "strong",
            "config": {"workload": "cluster LayerNorm (SURVEY §8f rank 3), PAPER.md:736 LN6 "
                                   "1152 x 65536 f32, one CTA cluster per row, DSM exchange",
                       "l2": "x, y 2 x 302 MB > L2"},
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": pk["hbm"],
                         "unit": "GB/s", "frac": round(gbs / pk["hbm"], 4),
                         "peak_source": f"{pk['src']} HBM copy bandwidth",
                         "algorithmic_bytes_per_launch": 8.0 * rows * n,
                         "traffic": traffic("layernorm_ln6") if ws == 1 else None},
            "clocks": clocks}


SIMP_BH, SIMP_S, SIMP_W1, SIMP_W2 = 16, 8192, 32, 512


def bench_simplicial(args, rank, ws, local):
    """2-simplicial attention forward, bf16 [16, 8192,
    128], windows w1=32 (K1) and w2=512 (K2), heads split across ranks.
    Algorithmic FLOP = 4*D per (i, j1, j2) triple (QK'.K2 + P.V2)."""
    import torch
    import paper_2605_10905_b200 as P
    from paper_2605_10905_b200 import shard
    L = P.lib()
    pk = peaks()
    dev = torch.device("cuda", local)
    r0, r1 = shard.head_shards(SIMP_BH, ws)[rank]
    bh = max(1, r1 - r0)
    g = torch.Generator(device=dev).manual_seed(31 + rank)
    t = [((torch.rand((bh, SIMP_S, 128), device=dev, generator=g) * 2 - 1).bfloat16())
         for _ in range(5)]
    o = torch.empty_like(t[0])
    lse = torch.empty((bh, SIMP_S), device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def step():
        P._check(L.mimw_b200_simplicial_attention_fwd(*(x.data_ptr() for x in t), o.data_ptr(),
                                                      lse.data_ptr(), bh, SIMP_S, 128, SIMP_W1,
                                                      SIMP_W2, 128 ** -0.5, sptr))

    steps = max(3, args.steps // 5)
    clk = Clocks(local)
    clk.start()
    secs = timed(step, steps, args.warmup, ws, stream)
    clocks = clk.stop()
    i = np.arange(SIMP_S, dtype=np.float64)
    triples = float(np.sum(np.minimum(SIMP_W1, i + 1) * np.minimum(SIMP_W2, i + 1)))
    flop_head = 4.0 * 128 * triples
    per = secs / steps
    achieved = flop_head * (r1 - r0) / per / 1e12
    return {"value": round(flop_head * SIMP_BH * steps / secs / 1e12, 2), "unit": "TFLOPS",
            "ms_per_step": round(per * 1e3, 4), "scaling": "strong",
            "config": {"workload": "2-simplicial attention fwd (SURVEY §8f rank 2), bf16 BH=16 "
                                   "S=8192 D=128, w1=32, w2=512",
                       "l2": "5 x 32 MiB inputs (K2/V2 windows re-read from L2 per K1 offset)"},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": pk["bf16"],
                         "unit": "TFLOP/s", "frac": round(achieved / pk["bf16"], 4),
                         "peak_source": f"{pk['src']} bf16 burst",
                         "algorithmic_flop_per_launch": flop_head * (r1 - r0),
                         "traffic": traffic("simplicial")},
            "clocks": clocks}


BWD_B, BWD_H, BWD_S = 4, 48, 8192  # PAPER.md:713 ABC4 (backward, non-causal, D=128)


def bench_attention_bwd(args, rank, ws, local):
    """attention backward, PAPER.md:713 ABC4 (B=4 H=48
    S=8192 D=128, non-causal), heads split across ranks; the non-causal
    forward (AFN4) timed on the same inputs.  FLOP: forward 4*S^2*D per head,
    backward 2.5x that (five S^2*D GEMMs)."""
    import torch
    import paper_2605_10905_b200 as P
    from paper_2605_10905_b200 import shard
    pk = peaks()
    dev = torch.device("cuda", local)
    r0, r1 = shard.head_shards(BWD_B * BWD_H, ws)[rank]
    bh = max(1, r1 - r0)
    g = torch.Generator(device=dev).manual_seed(13 + rank)
    q, k, v, do = ((torch.rand((1, bh, BWD_S, 128), device=dev, generator=g) * 2 - 1).bfloat16()
                   for _ in range(4))
    o, lse = P.attention_fwd(q, k, v, causal=False)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    stream = torch.cuda.current_stream()

    def fwd():
        P.attention_fwd(q, k, v, causal=False, out=o, lse=lse)

    def bwd():
        P.attention_bwd(q, k, v, o, do, lse, causal=False, dq=dq, dk=dk, dv=dv)

    steps = max(3, args.steps // 10)
    fsecs = timed(fwd, steps, args.warmup, ws, stream)
    clk = Clocks(local)
    clk.start()
    secs = timed(bwd, steps, args.warmup, ws, stream)
    clocks = clk.stop()
    fwd_flop_head = 4.0 * BWD_S * BWD_S * 128
    per = secs / steps
    achieved = 2.5 * fwd_flop_head * (r1 - r0) / per / 1e12
    return {"value": round(2.5 * fwd_flop_head * BWD_B * BWD_H * steps / secs / 1e12, 1),
            "unit": "TFLOPS", "ms_per_step": round(per * 1e3, 4), "scaling": "strong",
            "config": {"workload": "attention backward (SURVEY §8f rank 4), PAPER.md:713 ABC4 "
                                   "B=4 H=48 S=8192 D=128 non-causal, bf16, dQ by TMA reduce-add",
                       "l2": "Q, K, V, O, dO 5 x 384 MiB > L2"},
            "noncausal_fwd": {"value": round(fwd_flop_head * BWD_B * BWD_H * steps / fsecs / 1e12, 1),
                              "unit": "TFLOPS", "ms_per_step": round(fsecs / steps * 1e3, 4),
                              "workload": "PAPER.md:708 AFN4 B=4 H=48 S=8192 D=128 non-causal"},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": pk["bf16"],
                         "unit": "TFLOP/s", "frac": round(achieved / pk["bf16"], 4),
                         "peak_source": f"{pk['src']} bf16 burst",
                         "algorithmic_flop_per_launch": 2.5 * fwd_flop_head * (r1 - r0),
                         "traffic": traffic("attention_bwd")},
            "clocks": clocks}


MD_SHAPE = ("GD1", 8192, 2048, 16384)  # PAPER.md:751 multi-GPU GEMM shape (M, N, K)
NVLINK_GBS = 770.0  # B200_PROFILING.md: measured peer copy bandwidth per direction


def bench_multidevice(args, rank, ws, local):
    """the all-gather (K-gathered) multi-device GEMM,
    C = [A_0 | ... | A_{W-1}] . [B_0 ; ... ; B_{W-1}] with split s on device s
    (multi_device_gemm.mimw, oracles.cpp:57-80), PAPER.md:751 GD1 shape
    M=8192 N=2048 K=16384.  One process per GPU: each rank pulls the peers'
    splits over NVLink inside the GEMM kernel and computes its C row block.
    With one GPU the second device is emulated: its split lives in local HBM
    (standing in for the IPC-mapped peer buffer) and rank 0's launch is timed;
    the same launch is also timed as gather-then-GEMM (D2D copies + GEMM)."""
    import torch
    import paper_2605_10905_b200 as P
    from paper_2605_10905_b200 import multi_device as MD
    pk = peaks()
    dev = torch.device("cuda", local)
    name, m, n, k = MD_SHAPE
    world = ws if ws > 1 else 2
    ks = [k // world] * world
    rows = m // world
    g = torch.Generator(device=dev).manual_seed(23 + rank)
    stream = torch.cuda.current_stream()
    c = torch.empty((rows, n), device=dev, dtype=torch.bfloat16)
    flop_rank = 2.0 * rows * n * k
    remote_bytes = sum(2.0 * (rows * kk + kk * n) for kk in ks[1:])
    if ws > 1:
        ag = MD.AllGatherGemm(m, ks, n, device=dev)
        ag.a_local.copy_((torch.rand((m, ks[rank]), device=dev, generator=g) * 2 - 1).bfloat16())
        ag.b_local.copy_((torch.rand((ks[rank], n), device=dev, generator=g) * 2 - 1).bfloat16())
        torch.cuda.synchronize()
        barrier(ws)

        def step():
            ag(out=c)
        serial = None
    else:
        a = [(torch.rand((m, kk), device=dev, generator=g) * 2 - 1).bfloat16() for kk in ks]
        b = [(torch.rand((kk, n), device=dev, generator=g) * 2 - 1).bfloat16() for kk in ks]
        nb = MD.workspace_bytes(0, world, ks, rows, n)
        wsb = torch.empty(nb + 1024, device=dev, dtype=torch.uint8)
        wp = (wsb.data_ptr() + 1023) & ~1023
        ap_, bp_ = [t.data_ptr() for t in a], [t.data_ptr() for t in b]

        def step():
            MD.multi_device_gemm(0, world, ap_, bp_, ks, m, n, 0, rows, c.data_ptr(), n, wp, nb)
        a_land = torch.empty((rows, k), device=dev, dtype=torch.bfloat16)
        b_land = torch.empty((k, n), device=dev, dtype=torch.bfloat16)
        a_land[:, :ks[0]].copy_(a[0][:rows])
        b_land[:ks[0]].copy_(b[0])

        def serial_step():
            off = ks[0]
            for s_ in range(1, world):
                a_land[:, off:off + ks[s_]].copy_(a[s_][:rows])
                b_land[off:off + ks[s_]].copy_(b[s_])
                off += ks[s_]
            P.gemm(a_land, b_land, out=c)
        steps = max(10, args.steps)
        serial = timed(serial_step, steps, args.warmup, ws, stream) / steps
    steps = max(10, args.steps)
    clk = Clocks(local)
    clk.start()
    secs = timed(step, steps, args.warmup, ws, stream)
    clocks = clk.stop()
    per = secs / steps
    achieved = flop_rank / per / 1e12
    target = max(flop_rank / (pk["bf16"] * 1e12), remote_bytes / (NVLINK_GBS * 1e9))
    out = {"value": round(flop_rank * (ws if ws > 1 else 1) / per / 1e12, 1), "unit": "TFLOPS",
           "ms_per_step": round(per * 1e3, 4), "scaling": "strong" if ws > 1 else "weak",
           "config": {"workload": f"all-gather multi-device GEMM (SURVEY §8f rank 1), PAPER.md:751 "
                                  f"{name} M={m} N={n} K={k} bf16, K split over {world} devices, "
                                  f"C rows partitioned",
                      "devices": world,
                      "peers": "real (CUDA IPC over NVLink)" if ws > 1 else
                               "emulated: the second device's split in local HBM, rank 0 timed",
                      "comm": "comm warp in every GEMM CTA pair (library default)"},
           "roofline": {"bound": "tensor|nvlink", "achieved": round(achieved, 1), "peak": pk["bf16"],
                        "unit": "TFLOP/s", "frac": round(achieved / pk["bf16"], 4),
                        "target_ms": round(target * 1e3, 4),
                        "frac_of_target": round(target / per, 4),
                        "remote_bytes_per_rank": remote_bytes,
                        "target_rule": "max(FLOP / bf16 peak, remote bytes / 770 GB/s NVLink)",
                        "traffic": traffic("multi_device_gemm")},
           "clocks": clocks}
    if serial is not None:
        out["gather_then_gemm_ms"] = round(serial * 1e3, 4)
    if ws > 1:
        ag.close()
    return out


def torch_empty_cache():
    import torch
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="gemm", choices=["gemm", "attention", "fp8", "moe", "layernorm", "simplicial",
                             "multidevice", "attention_bwd", "launchcheck"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--fa-emu", type=int, default=-1, help="exp2 pairs of 8 on the FMA pipe")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        # every warm-up and timed step is one bounded row sample, sized so the
        # whole --steps K --warmup W run stays near 2 minutes
        per = min(12.0, max(1.0, 120.0 / (args.steps + args.warmup)))
        for _ in range(args.warmup):
            cpu_gemm_sample(per, single=False)
        vals, info = [], None
        for st in range(max(1, args.steps)):
            r = cpu_gemm_sample(per, single=(st == 0))
            info = info or r
            vals.append(r["value"])
        v = float(np.median(vals))
        fa = cpu_attention_sample()
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOPS",
               "n_gpus": int(os.environ.get("WORLD_SIZE", args.gpus)), "steps": len(vals),
               "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": "f32", "data": "synthetic U[-1,1] rounded to bf16",
               "config": {"workload": "configs[1] GEMM 8192^3 via reference oracle_gemm "
                                      "(oracles.cpp:14-26) on host cores, row-sampled"},
               "cpu_baseline": dict(info, value=v),
               "e2e": {"value": v, "unit": "TFLOPS", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0},
               "fa_fwd": {"value": fa["value"], "unit": "TFLOPS",
                          "config": {"workload": "configs[3] causal attention via reference oracle_attention "
                                                 "(oracles.cpp:119-145) on host cores, head-sampled"},
                          "cpu_baseline": fa}}
        print(json.dumps(out))
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    rank, ws, local = dist_init(args.gpus)
    fa = None
    if args.workload == "launchcheck":
        # the multi-rank launch path alone (no kernels): tests/test_bench_launch.py
        import torch.distributed as dist
        t = np.array([rank], dtype=np.int64)
        if ws > 1:
            import torch
            tt = torch.tensor([rank], dtype=torch.int64)
            dist.all_reduce(tt)
            t = tt.numpy()
        if rank == 0:
            print(json.dumps({"workload": "launchcheck", "n_gpus": ws, "rank_sum": int(t[0]),
                              "backend": dist.get_backend() if ws > 1 else None}))
        if ws > 1:
            dist.destroy_process_group()
        return
    if args.workload == "attention":
        res = bench_attention(args, rank, ws, local)
    elif args.workload == "fp8":
        res = bench_mxfp8(args, rank, ws, local)
    elif args.workload == "moe":
        res = bench_moe(args, rank, ws, local)
    elif args.workload == "layernorm":
        res = bench_layernorm(args, rank, ws, local)
    elif args.workload == "simplicial":
        res = bench_simplicial(args, rank, ws, local)
    elif args.workload == "multidevice":
        res = bench_multidevice(args, rank, ws, local)
    elif args.workload == "attention_bwd":
        res = bench_attention_bwd(args, rank, ws, local)
    else:
        res = bench_gemm(args, rank, ws, local)
        if not args.no_secondary:
            # each further workload starts after COOLDOWN_S idle seconds, so it
            # is not measured in the power / clock state the previous one left
            # behind (1 kW cap; e.g. LayerNorm read 3.9 instead of 5.4 TB/s
            # right after the MoE line)
            res["cooldown_s_between_workloads"] = COOLDOWN_S
            cooldown(ws)
            fa = bench_attention(args, rank, ws, local)
            torch_empty_cache()
            cooldown(ws)
            res["secondary"] = {"mxfp8_gemm": bench_mxfp8(args, rank, ws, local)}
            torch_empty_cache()
            cooldown(ws)
            moe = bench_moe(args, rank, ws, local)
            res["secondary"]["grouped_moe_gemm"] = {k: moe[k] for k in (
                "value", "unit", "ms_per_step", "scaling", "config", "roofline", "clocks",
                "reassembly")}
            torch_empty_cache()
            cooldown(ws)
            res["secondary"]["layernorm_cluster"] = bench_layernorm(args, rank, ws, local)
            cooldown(ws)
            res["secondary"]["simplicial_attention"] = bench_simplicial(args, rank, ws, local)
            torch_empty_cache()
            cooldown(ws)
            res["secondary"]["attention_bwd"] = bench_attention_bwd(args, rank, ws, local)
            torch_empty_cache()
            cooldown(ws)
            try:
                if ws > 1 and os.environ.get("MIMW_BENCH_MD", "1") == "0":
                    raise RuntimeError("disabled by MIMW_BENCH_MD=0")
                if ws > 1 and backend_for(ws) != "nccl":
                    # ranks sharing one GPU cannot meet in the device-side barrier
                    # (kernels of different processes do not run concurrently)
                    raise RuntimeError("skipped: ranks share a GPU (gloo functional run)")
                if ws > 1:
                    # real peers: a straggler is waited for at most this long (device-side barrier)
                    os.environ.setdefault("MIMW_PEER_WAIT_S", "60")
                res["secondary"]["multi_device_gemm"] = bench_multidevice(args, rank, ws, local)
            except Exception as e:  # never lose the headline line to the §8f extra
                res["secondary"]["multi_device_gemm"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0 and ws == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_attention_sample() if args.workload == "attention" else cpu_gemm_sample()
        if fa is not None:
            fa["cpu_baseline"] = cpu_attention_sample()
    if fa is not None:
        # FA-fwd (the other half of BASELINE's metric) as the LAST key of the
        # line, so it is in any captured tail of stdout
        res["fa_fwd"] = {k: fa[k] for k in ("value", "unit", "ms_per_step", "steps", "scaling", "config",
                                            "roofline", "clocks", "e2e", "cpu_baseline", "reassembly",
                                            "gpu_launches") if k in fa}
    if rank == 0:
        print(json.dumps(res))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
