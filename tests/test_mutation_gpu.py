"""Barrier-deletion (mutation) test of the default dense GEMM kernel, the GPU
form of the reference's acceptance test (acceptance.cpp:461-485): there, every
barrier_wait of gemm_pipeline.mimw is deleted in turn and the simulator must
notice (race, failure or rel_error > 1e-4) within 100 SeededRandom schedules.

Here each mbarrier wait of the wide-tile kernel (gemm_wide.cuh, WIDE_WAIT tags)
is deleted in a test build (paper_2605_10905_b200/build.py: build_mutant, ~1 s
watchdog) that also perturbs the schedule (MIMW_PERTURB: random 0.5-16.5 us
sleeps in the epilogue and the CLC issuer, the stand-in for SeededRandom), and
the mutant runs the GEMM on five shapes, three times each, in a subprocess.
Detected = wrong or unwritten outputs, a CUDA error (the watchdog's trap
included) or a timeout.  The unmutated, perturbed builds must pass the same
check, so the check and the perturbation are sound.

Wait 13 (the CLC issuer waiting for every consumer to release a response slot)
cannot fire with the shipped 4-slot ring: waits 1-3 already bound the issuer's
lead over the slowest consumer to 3 tile ids (reaching id u needs the MMA on
u-1, hence the epilogue done draining u-2, hence done with u-3).  Its mutant is
therefore built with a 2-slot ring, where the lead can exceed the ring."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "mutants", "_build")
CHECK = os.path.join(ROOT, "tests", "mutants", "check_gemm.py")
# tag -> (the wait it deletes (gemm_wide.cuh), CLC ring slots of the build)
WAITS = {
    1: ("producer waits for a ring slot to be freed by the MMA commit (empty)", 4),
    2: ("MMA waits for the epilogue to drain the accumulator (tmem empty)", 4),
    3: ("MMA waits for a stage's TMA bytes (full)", 4),
    4: ("epilogue waits for the tile's last MMA commit (tmem full)", 4),
    12: ("tile-id consumers wait for the CLC response", 4),
    13: ("CLC issuer waits for every consumer to release a response slot", 2),
}
CONTROLS = (4, 2)  # unmutated + perturbed builds, one per ring size


@pytest.fixture(scope="module")
def libs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available to build the mutants")
    from paper_2605_10905_b200 import build
    build.build()
    jobs = [(t, slots) for t, (_, slots) in WAITS.items()] + [(0, s) for s in CONTROLS]
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        out = list(ex.map(lambda j: build.build_mutant(j[0], OUT, clc_slots=j[1]), jobs))
    return dict(zip(jobs, out))


def _run(lib):
    env = dict(os.environ, MIMW_B200_LIB=lib)
    try:
        r = subprocess.run([sys.executable, CHECK], capture_output=True, text=True, timeout=240, env=env)
    except subprocess.TimeoutExpired:
        return "detected: timeout"
    out = (r.stdout.strip().splitlines() or [""])[-1]
    if r.returncode != 0:
        return f"detected: exit {r.returncode}: {(r.stderr.strip().splitlines() or [''])[-1][:200]}"
    return out


def test_product_build_passes_the_check():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_10905_b200 import build
    assert _run(build.build()) == "ok"


@pytest.mark.parametrize("slots", CONTROLS)
def test_perturbed_unmutated_build_passes_the_check(libs, slots):
    assert _run(libs[(0, slots)]) == "ok"


@pytest.mark.parametrize("tag", sorted(WAITS))
def test_deleting_a_wait_is_detected(libs, tag):
    what, slots = WAITS[tag]
    res = _run(libs[(tag, slots)])
    print(f"wait {tag} ({what}, {slots}-slot ring): {res}")
    assert res.startswith("detected"), f"deleting wait {tag} ({what}) went undetected"
