"""Regenerate a golden case's inputs (seed rule of case.cpp:82-92) and load
its reference outputs (MIMWTNSR, tensor_io.cpp:30-78)."""
import os

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_inputs(case):
    if "seeds" in case:  # explicit per-input seeds (collective_dot)
        xs = {n: oracle.random_tile(s, case["seeds"][n]) for n, s in case["inputs"]}
    else:
        xs = oracle.make_inputs({n: s for n, s in case["inputs"]}, case["seed"])
    if case.get("bf16"):
        xs = {n: oracle.round_bf16(x) for n, x in xs.items()}
    return xs


def case_outputs(case):
    return {n: oracle.read_tensor(os.path.join(GOLDEN, f)) for n, f in case["outputs"].items()}
