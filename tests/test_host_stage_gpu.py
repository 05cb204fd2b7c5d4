"""The host-Tile GEMM entries round f32 -> bf16 on the host threads
(csrc/host_stage.cu, MIMW_HOST_STAGE=1, default) instead of in device staging
kernels (MIMW_HOST_STAGE=0).  Both must give bit-identical C, including
signed zeros, denormals, values that round up to Inf, Inf and NaN inputs,
ragged shapes (K / N padding) and the K-concatenated multi-part entry
(oracle_multi_device_gemm, oracles.cpp:57-80).  The knob is read once per
process, so each arm runs in its own interpreter."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2605_10905_b200 as P
out = {}
def pin(x):
    # pinned host inputs: the staging modes 2 / 3 DMA f32 chunks straight from
    # them (pageable inputs always take the all-host-rounding path)
    if os.environ.get("MIMW_TEST_PINNED") != "1":
        return x
    import torch
    t = torch.empty(x.shape, dtype=torch.float32).pin_memory()
    t.numpy()[...] = x
    return t.numpy()
rng = np.random.default_rng(7)
for m, k, n in [(1, 1, 1), (37, 29, 45), (300, 200, 264), (1500, 136, 520), (3000, 1100, 72)]:
    a = (rng.standard_normal((m, k)) * 3).astype(np.float32)
    b = (rng.standard_normal((k, n)) * 3).astype(np.float32)
    flat = a.reshape(-1)
    specials = np.array([0.0, -0.0, 1e-40, -3e-39, 3.3895314e38, -3.3895314e38, 1.0000001, 1.00390625,
                         1.01171875, np.inf, -np.inf, np.nan], np.float32)
    flat[:min(len(flat), len(specials))] = specials[:len(flat)]
    a, b = pin(a), pin(b)
    out[f"g{m}_{k}_{n}"] = P.oracle_gemm(a, b)
    a1 = (rng.standard_normal((m, 24)) * 2).astype(np.float32)
    b1 = (rng.standard_normal((24, n)) * 2).astype(np.float32)
    out[f"md{m}_{k}_{n}"] = P.oracle_multi_device_gemm(a, pin(a1), b, pin(b1))
np.savez(sys.argv[2], **out)
'''


def _run(tmp_path, flag, pinned=True):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    path = str(tmp_path / f"arm{flag}_{int(pinned)}.npz")
    env = dict(os.environ, MIMW_HOST_STAGE=str(flag), MIMW_TEST_PINNED="1" if pinned else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, path], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


@pytest.mark.parametrize("mode,pinned", [(1, True), (2, True), (3, True), (3, False)])
def test_host_staging_bit_identical_to_device_staging(tmp_path, mode, pinned):
    """mode 1: all rounding on the host; 2: B's odd row chunks and all of A
    rounded on the device; 3: odd chunks of both on the device.  Pageable
    buffers (pinned=False): all-host rounding and C through pinned slots."""
    host, dev = _run(tmp_path, mode, pinned), _run(tmp_path, 0)
    assert sorted(host.files) == sorted(dev.files)
    for name in host.files:
        x, y = host[name], dev[name]
        assert x.shape == y.shape, name
        same = (x.view(np.uint32) == y.view(np.uint32)) | (np.isnan(x) & np.isnan(y))
        assert same.all(), (name, int((~same).sum()))
