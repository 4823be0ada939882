"""CPU model of the fused kernel's scheduling protocol (csrc/fused.cuh,
tools/fused_sim.py): under random interleavings of CTAs every job runs exactly
once, after its dependency is counted, and the ticket protocol never
deadlocks (a CTA blocks only while holding no unfinished job)."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def model():
    spec = importlib.util.spec_from_file_location("fused_sim", os.path.join(ROOT, "tools", "fused_sim.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_protocol_exactly_once_no_deadlock(model):
    for args in model.CASES:
        for seed in range(4):
            assert model.sim(*args, seed) == "ok", (args, seed)
