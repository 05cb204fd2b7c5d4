"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference oracles (oracle/_ref/libmimw_ref.so, built by
oracle/Makefile from /root/reference/proj/core/src) on the reference's own
seeded cases and writes outputs in the reference's MIMWTNSR format
(tensor_io.cpp:30-48), plus ``manifest.json`` describing how each input is
regenerated (seed rule of case.cpp:82-92, optional bf16 rounding).

Cases (reference pins from SURVEY.md §8c):
  gemm_pipeline      kernels/gemm_pipeline.case        seed 7,  tol 1e-4
  gemm_clc           kernels/gemm_clc.case             seed 19, tol 1e-4
  multi_device_gemm  kernels/multi_device_gemm.case    seed 23, tol 1e-4
  simplicial_attn    kernels/simplicial_attention.case seed 31, tol 1e-3
  attention_degen    tests/acceptance.cpp:333-355      seed 31, tol 1e-4
  collective_dot     tests/acceptance.cpp:392-421      seeds 41/42
  layernorm_cluster  kernels/layernorm_cluster.case    seed 5,  tol 1e-5
plus bf16-rounded GPU-parity cases at kernel tile scale (north_star: bf16
within rel-err 1e-2).

Run here (needs /root/reference):  python tests/golden/make_golden.py
"""
import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

R = oracle.REF
if R is None:
    sys.exit("oracle/_ref not built (needs /root/reference): run make -C oracle")


def rt(shape, seed):
    """reference random_tile."""
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    arr = (ctypes.c_int64 * len(shape))(*shape)
    R.ref_random_tile(arr, len(shape), seed, out)
    return out.reshape(shape)


def inputs(spec, seed, bf16=False):
    out = {}
    for k, (name, shape) in enumerate(spec):
        x = rt(shape, seed * 1000003 + k)
        out[name] = oracle.round_bf16(x) if bf16 else x
    return out


def wt(name, x):
    x = np.ascontiguousarray(x, np.float32)
    shape = (ctypes.c_int64 * max(1, x.ndim))(*x.shape)
    assert R.ref_write_tensor(os.path.join(HERE, name).encode(), x.ravel(), shape, x.ndim) == 0
    return name


def ref_gemm(a, b):
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), np.float32)
    R.ref_oracle_gemm(np.ascontiguousarray(a), np.ascontiguousarray(b), c, m, n, k)
    return c


def ref_attn(q, k, v, w, scale):
    s, d = q.shape
    o = np.empty((s, d), np.float32)
    R.ref_oracle_attention(q, k, v, o, s, d, w, scale)
    return o


def ref_simplicial(q, k1, v1, k2, v2, w1, w2, scale):
    s, d = q.shape
    o = np.empty((s, d), np.float32)
    lse = np.empty(s, np.float32)
    R.ref_oracle_simplicial_attention(q, k1, v1, k2, v2, o, lse, s, d, w1, w2, scale)
    return o, lse


def main():
    man = []

    def gemm_case(name, seed, m, k, n, tol, bf16=False, source=""):
        spec = [("a", [m, k]), ("b", [k, n])]
        x = inputs(spec, seed, bf16)
        man.append(dict(name=name, oracle="gemm", seed=seed, inputs=spec, bf16=bf16,
                        tolerance=tol, source=source,
                        outputs={"c": wt(f"{name}.c.tnsr", ref_gemm(x["a"], x["b"]))}))

    gemm_case("gemm_pipeline", 7, 64, 64, 64, 1e-4, source="kernels/gemm_pipeline.case:1-7")
    gemm_case("gemm_clc", 19, 64, 128, 64, 1e-4, source="kernels/gemm_clc.case:1-7")

    # multi_device_gemm: inputs a0 a1 b0 b1 (multi_device_gemm.mimw:7-10)
    spec = [("a0", [64, 64]), ("a1", [64, 64]), ("b0", [64, 32]), ("b1", [64, 32])]
    x = inputs(spec, 23)
    c = np.empty((64, 32), np.float32)
    R.ref_oracle_multi_device_gemm(x["a0"], x["a1"], x["b0"], x["b1"], c, 64, 64, 64, 32)
    man.append(dict(name="multi_device_gemm", oracle="multi_device_gemm", seed=23, inputs=spec,
                    bf16=False, tolerance=1e-4, source="kernels/multi_device_gemm.case:1-8",
                    outputs={"c": wt("multi_device_gemm.c.tnsr", c)}))

    # simplicial attention (simplicial_attention.mimw:8-12) and its degeneration
    spec = [(n_, [32, 16]) for n_ in ("q", "k1", "v1", "k2", "v2")]
    x = inputs(spec, 31)
    o, lse = ref_simplicial(x["q"], x["k1"], x["v1"], x["k2"], x["v2"], 2, 16, 0.25)
    man.append(dict(name="simplicial_attention", oracle="simplicial_attention", seed=31,
                    inputs=spec, bf16=False, tolerance=1e-3,
                    scalars={"w1": 2, "w2": 16, "scale": 0.25},
                    source="kernels/simplicial_attention.case:1-10",
                    outputs={"o": wt("simplicial_attention.o.tnsr", o),
                             "lse": wt("simplicial_attention.lse.tnsr", lse)}))
    ones = np.ones((32, 16), np.float32)
    o1, _ = ref_simplicial(x["q"], ones, ones, x["k2"], x["v2"], 1, 16, 0.25)
    o2 = ref_attn(x["q"], x["k2"], x["v2"], 16, 0.25)
    assert R.ref_rel_error(o1.ravel(), o2.ravel(), o1.size) <= 1e-4
    man.append(dict(name="attention_degeneration", oracle="attention", seed=31, inputs=spec,
                    bf16=False, tolerance=1e-4, scalars={"w": 16, "scale": 0.25},
                    map={"q": "q", "k": "k2", "v": "v2"},
                    source="tests/acceptance.cpp:333-355",
                    outputs={"o": wt("attention_degeneration.o.tnsr", o2)}))

    # collective_dot: a = random_tile({32,16}, 41), b = random_tile({16,24}, 42)
    a, b = rt([32, 16], 41), rt([16, 24], 42)
    man.append(dict(name="collective_dot", oracle="gemm", seeds={"a": 41, "b": 42},
                    inputs=[("a", [32, 16]), ("b", [16, 24])], bf16=False, tolerance=1e-4,
                    source="tests/acceptance.cpp:392-421",
                    outputs={"c": wt("collective_dot.c.tnsr", ref_gemm(a, b))}))

    # layernorm_cluster (x w b, eps 1e-5)
    spec = [("x", [4, 1024]), ("w", [1024]), ("b", [1024])]
    x = inputs(spec, 5)
    y = np.empty((4, 1024), np.float32)
    mu = np.empty(4, np.float32)
    rs = np.empty(4, np.float32)
    R.ref_oracle_layernorm(x["x"], x["w"], x["b"], 1e-5, y, mu, rs, 4, 1024)
    man.append(dict(name="layernorm_cluster", oracle="layernorm", seed=5, inputs=spec,
                    bf16=False, tolerance=1e-5, scalars={"eps": 1e-5},
                    source="kernels/layernorm_cluster.case:1-9",
                    outputs={"y": wt("layernorm_cluster.y.tnsr", y)}))

    # random_tile determinism vector (tests/test_kernels.cpp:74-81)
    man.append(dict(name="random_tile_9", oracle="random_tile", seeds={"x": 9}, inputs=[("x", [64])],
                    bf16=False, tolerance=0, source="tests/test_kernels.cpp:74-81",
                    outputs={"x": wt("random_tile_9.x.tnsr", rt([64], 9))}))

    # ---- bf16 GPU-parity cases (north_star: bf16 within 1e-2) ----
    gemm_case("gemm_bf16_256x320x384", 7, 256, 320, 384, 1e-2, bf16=True,
              source="north_star bf16 GEMM; seed rule case.cpp:88")
    gemm_case("gemm_bf16_ragged_200x136x72", 19, 200, 136, 72, 1e-2, bf16=True,
              source="ragged edges (not tile multiples)")
    for nm, s, w in (("attention_bf16_causal_s256", 256, 256),
                     ("attention_bf16_window_s320_w100", 320, 100)):
        spec = [("q", [s, 128]), ("k", [s, 128]), ("v", [s, 128])]
        x = inputs(spec, 31, bf16=True)
        scale = 1.0 / np.sqrt(128.0)
        o = ref_attn(x["q"], x["k"], x["v"], w, scale)
        man.append(dict(name=nm, oracle="attention", seed=31, inputs=spec, bf16=True,
                        tolerance=1e-2, scalars={"w": w, "scale": scale},
                        map={"q": "q", "k": "k", "v": "v"},
                        source="oracles.cpp:119-145 at D=128",
                        outputs={"o": wt(f"{nm}.o.tnsr", o)}))

    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(man, f, indent=1)
    print(f"wrote {len(man)} golden cases")


if __name__ == "__main__":
    main()
