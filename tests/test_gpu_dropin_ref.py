"""The reference's own harness driving the GPU drop-in.

* oracle/_ref/acceptance_dropin: the reference's acceptance gate
  (tests/acceptance.cpp) with its harness sources (src/verify.cpp, oracle.cpp,
  bench.cpp), compiled UNCHANGED against the drop-in headers include/pafft/*.hpp
  and linked to libpafft_b200.so (oracle/Makefile).  Criteria 1-5 (oracle
  equivalence over the verification grid, bitwise decomposition, involution,
  reordering-pass accounting), 8 (cost models) and 9 (1000 + 1000 random
  shapes: Parseval and linearity at 1e-10) must PASS, every transform and
  convolution running on the B200.  Criteria 6 and 7 time the host-buffer
  path (PCIe copies dominate both sides) and are reported, not gated; the
  reference itself fails 7 (proj/test_output.txt).
* oracle/_ref/unit_dropin: the reference's doctest unit tests
  (tests/test_{core,permutation,butterfly,transform,convolution,oracle,bench}.cpp),
  compiled unchanged against the drop-in headers with a minimal
  doctest-compatible runner (oracle/doctest_shim/doctest.h); every assertion
  must pass except the intended behaviour changes listed in INTENDED_UNIT.
* oracle/_ref/test_smoke.py: the reference's Python smoke test, unchanged,
  through a `pafft` alias of the product package (tests/refsmoke/); the radix-3
  rejection (test_smoke.py:70) is the one intended break, marked xfail.

Both artefacts are built in the container from /root/reference and travel
with the repo; the tests skip when they were never built.
"""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
GATED = {1, 2, 3, 4, 5, 8, 9}
# assertions of the reference's unit tests that this build changes on purpose
INTENDED_UNIT = {
    "test_core.cpp:17": "radix_from_value(3) is accepted: radix 3 and 5 are supported (BASELINE configs 2 and 5)",
}


def test_reference_acceptance_gate_on_gpu():
    exe = os.path.join(REF, "acceptance_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/acceptance_dropin not built (reference sources absent at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout
    print(out)
    print(r.stderr[-3000:], file=sys.stderr)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "acceptance_dropin.log"), "w") as f:
        f.write(out + "\n--- stderr ---\n" + r.stderr)
    got = {}
    for line in out.splitlines():
        m = re.match(r"\[(PASS|FAIL)\] (\d+)\. ", line)
        if m:
            got[int(m.group(2))] = m.group(1)
    assert sorted(got) == list(range(1, 10)), out
    failed = [c for c in sorted(GATED) if got[c] != "PASS"]
    assert not failed, f"criteria {failed} failed:\n{out}\n{r.stderr[-3000:]}"


def test_reference_unit_tests_on_gpu():
    exe = os.path.join(REF, "unit_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/unit_dropin not built (reference sources absent at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout
    print(out[-4000:])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "unit_dropin.log"), "w") as f:
        f.write(out + "\n--- stderr ---\n" + r.stderr)
    assert "[doctest-shim] test cases:" in out, out[-3000:] + r.stderr[-2000:]
    failed = {}
    for line in out.splitlines():
        m = re.match(r"FAILED (\S+):(\d+): (.*)", line)
        if m:
            failed[os.path.basename(m.group(1)) + ":" + m.group(2)] = m.group(3)
    unexpected = {k: v for k, v in failed.items() if k not in INTENDED_UNIT}
    assert not unexpected, unexpected
    assert set(failed) == set(INTENDED_UNIT), f"intended changes not observed: {set(INTENDED_UNIT) - set(failed)}"
    cases = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert cases and int(cases.group(1)) >= 55, out[-2000:]


def test_reference_python_smoke_through_alias():
    smoke = os.path.join(REF, "test_smoke.py")
    if not os.path.exists(smoke):
        pytest.skip("oracle/_ref/test_smoke.py not staged (reference sources absent at build time)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refsmoke"), ROOT, env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", smoke, "-q", "-p", "refsmoke_plugin", "-p", "no:cacheprovider",
                        "--rootdir", REF, "-c", os.devnull],
                       capture_output=True, text=True, timeout=600, cwd=REF, env=env)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert re.search(r"\b\d+ passed", r.stdout) and "1 xfailed" in r.stdout, r.stdout[-2000:]
