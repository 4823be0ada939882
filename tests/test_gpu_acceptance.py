"""GPU analogue of the reference's acceptance criterion 6 (convolution speedup
at scale, tests/acceptance.cpp:160-205): the permutation-free
convolution must beat the standard-order one at radix 4, n = 2^20, 2^22,
2^24 (the reference requires ratio >= 1, targets >= 1.2 at 2^22).  Timed with
CUDA events through bench_ops (the reference's bench op table on the GPU) at
a fixed 2^24 points per timed call, so small sizes still fill the GPU.
Measured on B200: 2.9x / 2.8x / 2.3x (profiles/r01_bench_ops_table.md)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("log2n", [20, 22, 24])
def test_permfree_beats_standard_order(log2n):
    from paper_2506_12718_b200 import bench_ops
    n = 1 << log2n
    batch = max(1, (1 << 24) // n)
    std = bench_ops.run("conv-std", 4, [n], batch, reps=5)  # also checks both pipelines agree
    pa = bench_ops.run("conv-pa", 4, [n], batch, reps=5)
    ratio = std["median_s"] / pa["median_s"]
    print(f"n=2^{log2n} batch={batch} conv-std/conv-pa = {ratio:.3f}")
    assert ratio >= 1.2, ratio
    assert pa["timed_permutation_passes"] == 0 and std["timed_permutation_passes"] == 2 * batch * 5
