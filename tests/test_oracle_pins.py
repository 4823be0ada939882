"""Pins the oracle (oracle/pafft_oracle.c, the CPU restatement) before it is
trusted as the GPU checker:

* the known-answer values of the reference's own unit tests
  (test_butterfly.cpp:28-45, test_convolution.cpp:22-61/63-79,
  test_core.cpp:44-70, test_permutation.cpp:15-77, test_oracle.cpp);
* golden vectors produced by the reference library itself
  (tests/golden/reference_golden.npz, made by tests/golden/make_golden.py from
  oracle/_ref, i.e. pafft compiled from its own sources);
* pafft's radix-agnostic direct O(N^2) sums for radix 3 and 5, which pafft's
  ladders cannot run (core.hpp:14-19);
* live agreement with oracle/_ref where it is present.
CPU only.
"""
import os

import numpy as np
import pytest

from helpers import convolution_tolerance, max_diff, rand_c, rel_l2, transform_tolerance

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN)


def _cases(gold):
    keys = sorted({k.rsplit("_", 1)[0] for k in gold.files})
    out = []
    for k in keys:
        r, d = k.split("_")
        out.append((int(r[1:]), [int(v) for v in d.split("x")], k))
    return out


# ----------------------------------------------------------- known answers
def test_four_point_ladders(orc):
    """test_butterfly.cpp:28-45."""
    p = orc.plan(2, [4])
    import oracle
    assert max_diff(p.butterfly_line(np.array([1, 3, 2, 4], complex), 0, oracle.FORWARD),
                    [10, -2 + 2j, -2, -2 - 2j]) < 1e-13
    assert max_diff(p.butterfly_line(np.array([10, -2, -2 + 2j, -2 - 2j]), 0, oracle.CONJUGATE),
                    [4, 8, 12, 16]) < 1e-13
    assert max_diff(p.butterfly_line(np.array([1, 2, 3, 4], complex), 0, oracle.TRANSPOSED),
                    [10, -2, -2 + 2j, -2 - 2j]) < 1e-13


def test_filter_preparation_and_delay(orc):
    """test_convolution.cpp:32-61."""
    p = orc.plan(2, [4])
    assert np.array_equal(p.prepare_filter(np.array([0, 1, 2, 3], complex)), np.array([0, 2, 1, 3], complex))
    g = p.filter_from_impulse(np.array([0, 1, 0, 0], complex))
    assert max_diff(g, [1, -1j, -1, 1j]) < 1e-14
    x = np.array([1, 2, 3, 4], complex)
    assert max_diff(p.convolve_standard(x, g), [4, 1, 2, 3]) < 1e-13
    assert max_diff(p.convolve_permfree(x, p.prepare_filter(g)), [4, 1, 2, 3]) < 1e-13
    # pointwise multiply (test_convolution.cpp:22-30) through a 1-point plan
    assert max_diff(orc.plan(2, [1]).convolve_permfree(np.array([1 + 2j]), np.array([3 + 4j])), [-5 + 10j]) == 0


def test_pass_accounting(orc):
    """test_convolution.cpp:63-79: standard 2, prepare 1, permfree 0."""
    p = orc.plan(4, [16, 16])
    g, x = rand_c(256, 73), rand_c(256, 74)
    orc.reset_pass_count()
    p.convolve_standard(x, g)
    assert orc.pass_count() == 2
    orc.reset_pass_count()
    gh = p.prepare_filter(g)
    assert orc.pass_count() == 1
    orc.reset_pass_count()
    p.convolve_permfree(x, gh)
    assert orc.pass_count() == 0


def test_digit_reverse_and_maps(orc):
    """test_permutation.cpp:15-31 and test_core.cpp:44-70."""
    assert orc.digit_reverse(6, 2, 3) == 3
    assert orc.digit_reverse(5, 4, 2) == 5
    assert orc.digit_reverse(0, 8, 4) == 0
    assert orc.digit_reverse(1, 2, 3) == 4
    assert orc.digit_reverse(7, 8, 1) == 7
    assert orc.digit_reverse(5, 3, 2) == 7  # (1,2)_3 -> (2,1)_3, SURVEY.md 4
    import oracle
    for bad in [(8, 2, 3), (1, 2, 0)]:
        with pytest.raises(oracle.OracleError):
            orc.digit_reverse(*bad)
    p = orc.plan(2, [8])
    x = np.arange(8).astype(complex)
    assert np.array_equal(p.permute(x).real, [0, 4, 2, 6, 1, 5, 3, 7])
    assert np.array_equal(orc.plan(4, [4]).permute(np.arange(4).astype(complex)).real, [0, 1, 2, 3])


def test_plan_validation(orc):
    """test_core.cpp:29-42 (plus radix 3/5 now legal, 7 still not)."""
    import oracle
    for radix, dims, code in [(2, [], 2), (8, [4], 1), (4, [8], 1), (2, [0], 1), (2, [8, 3], 1), (7, [49], 7)]:
        with pytest.raises(oracle.OracleError) as e:
            orc.plan(radix, dims)
        assert e.value.code == code
    orc.plan(3, [9])
    orc.plan(5, [25, 5])


def test_permutation_involution_and_sweeps(orc):
    """test_permutation.cpp:39-77, 297-331."""
    for radix, dims in [(2, [64, 64]), (4, [64, 16]), (8, [4096]), (2, [16, 16, 16]), (3, [27, 9]), (5, [25, 5, 5])]:
        p = orc.plan(radix, dims)
        x = rand_c(p.total, 23)
        y = p.permute(x)
        assert np.array_equal(np.sort(y.real), np.sort(x.real))
        assert np.array_equal(p.permute(y), x)
        # Kronecker rule: out(i1..id) = in(rev(i1)..rev(id))
        revs = [np.array([orc.digit_reverse(j, radix, round(np.log(n) / np.log(radix))) for j in range(n)])
                for n in dims]
        xt = x.reshape(dims[::-1])
        want = xt
        for ax, r in enumerate(revs):
            want = np.take(want, r, axis=len(dims) - 1 - ax)
        assert np.array_equal(y, want.reshape(-1))


def test_twiddle_tables(orc):
    """test_core.cpp:72-99: |w| = 1, w[j] w[n-j] = 1, stage rule."""
    import ctypes as C
    for n in (8, 64, 4096, 2187, 3125):
        radix = 2 if n in (8, 64, 4096) else (3 if n == 2187 else 5)
        p = orc.plan(radix, [n])
        st = p.ptr.contents
        re = np.ctypeslib.as_array(st.tw_re[0], shape=(n,))
        im = np.ctypeslib.as_array(st.tw_im[0], shape=(n,))
        w = re + 1j * im
        assert w[0] == 1
        assert np.abs(np.abs(w) - 1).max() < 1e-15
        assert np.abs(w[1:] * w[:0:-1] - 1).max() < 1e-14
        assert np.abs(w - np.exp(-2j * np.pi * np.arange(n) / n)).max() < 1e-13
    del C


def test_naive_oracles(orc):
    """test_oracle.cpp: 4-point DFT, impulse/flat pairs, backward inverts forward."""
    assert max_diff(orc.naive_dft(np.array([1, 2, 3, 4], complex), [4]), [10, -2 + 2j, -2, -2 - 2j]) < 1e-13
    d = np.zeros(8, complex)
    d[0] = 1
    assert max_diff(orc.naive_dft(d, [8]), np.ones(8)) < 1e-13
    x = rand_c(16, 11)
    assert max_diff(orc.naive_dft(orc.naive_dft(x, [16]), [16], backward=True), x) < 1e-12


# ----------------------------------------------------------- golden vectors
def test_golden_radix_248_bit_level(orc, gold):
    """The restatement against pafft's own outputs (radix 2/4/8)."""
    n_checked = 0
    for radix, dims, key in _cases(gold):
        if radix not in (2, 4, 8):
            continue
        x, h = gold[key + "_x"], gold[key + "_h"]
        p = orc.plan(radix, dims)
        n = p.total
        g = p.filter_from_impulse(h)
        assert rel_l2(g, gold[key + "_g"]) <= 1e-15
        ghat = p.prepare_filter(gold[key + "_g"])
        assert np.array_equal(ghat, gold[key + "_ghat"])  # pure data movement: bit-exact
        assert np.array_equal(p.permute(x), gold[key + "_permuted"])
        yp = p.convolve_permfree(x, gold[key + "_ghat"])
        ys = p.convolve_standard(x, gold[key + "_g"])
        assert rel_l2(yp, gold[key + "_permfree"]) <= 1e-14
        assert rel_l2(ys, gold[key + "_standard"]) <= 1e-14
        import oracle
        for v, name in [(oracle.TRANSPOSED, "transposed"), (oracle.FORWARD, "forward"),
                        (oracle.CONJUGATE, "conjugate")]:
            assert rel_l2(p.butterfly_tensor(x, v), gold[key + "_" + name]) <= 1e-14
        if radix == 2:  # radix 2: the generic combine is exactly the reference's
            assert np.array_equal(yp, gold[key + "_permfree"])
        if key + "_direct" in gold.files:
            tol = convolution_tolerance(n, np.abs(x).max(), np.abs(h).max())
            assert max_diff(yp, gold[key + "_direct"]) <= tol
        n_checked += 1
    assert n_checked >= 15


def test_golden_radix_35_against_reference_direct_sum(orc, gold):
    """Radix 3/5 pipelines against pafft's direct sum and naive DFT."""
    n_checked = 0
    for radix, dims, key in _cases(gold):
        if radix not in (3, 5):
            continue
        x, h = gold[key + "_x"], gold[key + "_h"]
        p = orc.plan(radix, dims)
        n = p.total
        g = p.filter_from_impulse(h)
        assert rel_l2(g, gold[key + "_dft"]) <= 1e-13
        yp = p.convolve_permfree(x, p.prepare_filter(g))
        ys = p.convolve_standard(x, g)
        direct = gold[key + "_direct"]
        tol = convolution_tolerance(n, np.abs(x).max(), np.abs(h).max())
        assert max_diff(yp, direct) <= tol and max_diff(ys, direct) <= tol
        assert rel_l2(yp, direct) <= 1e-13
        assert rel_l2(yp, ys) <= 1e-13
        n_checked += 1
    assert n_checked >= 10


def test_oracle_matches_numpy_at_moderate_size(orc):
    for radix, dims in [(3, [3 ** 9]), (5, [5 ** 6]), (2, [1 << 14]), (4, [64, 64]), (3, [81, 243])]:
        n = int(np.prod(dims))
        x, h = rand_c(n, 5), rand_c(n, 6)
        p = orc.plan(radix, dims)
        y = p.convolve_permfree(x, p.prepare_filter(p.filter_from_impulse(h)))
        shp = dims[::-1]
        ref = np.fft.ifftn(np.fft.fftn(x.reshape(shp)) * np.fft.fftn(h.reshape(shp))).reshape(-1)
        assert rel_l2(y, ref) <= 1e-14


def test_oracle_transform_tolerance_grid(orc):
    """verify.cpp:76-100 restated: ladder o reversal = DFT on the grid <= 4096."""
    from helpers import GRID, GRID_ODD
    for radix, dims in GRID + GRID_ODD:
        n = int(np.prod(dims))
        if n > 4096:
            continue
        x = rand_c(n, 31 + n)
        p = orc.plan(radix, dims)
        want = orc.naive_dft(x, dims)
        assert max_diff(p.fft_forward(x), want) <= transform_tolerance(n, np.abs(x).max()) * 2
        assert max_diff(p.permute(p.butterfly_tensor(x, 2)), want) <= transform_tolerance(n, np.abs(x).max()) * 2


def test_live_reference_agreement(orc, ref):
    """Where oracle/_ref exists: the restatement equals pafft on fresh inputs."""
    for radix, dims in [(2, [2048]), (4, [16, 64]), (8, [8, 64]), (2, [4, 4, 8]), (4, [4, 4, 4, 4])]:
        n = int(np.prod(dims))
        x, h = rand_c(n, 41), rand_c(n, 42)
        po, pr = orc.plan(radix, dims), ref.plan(radix, dims)
        go, gr = po.filter_from_impulse(h), pr.filter_from_impulse(h)
        assert rel_l2(go, gr) <= 1e-15
        assert rel_l2(po.convolve_permfree(x, po.prepare_filter(go)),
                      pr.convolve_permfree(x, pr.prepare_filter(gr))) <= 1e-15


# ------------------------------------------------------ per-axis radices
def _rev(j, r, n):
    o = 0
    while n > 1:
        o, j, n = o * r + j % r, j // r, n // r
    return o


def test_mixed_radix_oracle_pins(orc):
    """a different radix per axis.  Pinned by pafft's
    radix-agnostic direct sum and naive DFT (oracle.cpp:50-123 restated), by
    numpy, by the per-axis digit reversal of the prepared filter, and by the
    uniform-radix plan when all radices agree."""
    from helpers import GRID_MIXED
    for radices, dims in GRID_MIXED:
        n = int(np.prod(dims))
        x, h = rand_c(n, 71 + n), rand_c(n, 72 + n)
        p = orc.plan(radices, dims)
        g = p.filter_from_impulse(h)
        if n <= 4096:
            assert max_diff(g, orc.naive_dft(h, dims)) <= transform_tolerance(n, np.abs(h).max()) * 2
            direct = orc.naive_conv(x, h, dims)
        else:
            shp = dims[::-1]
            direct = np.fft.ifftn(np.fft.fftn(x.reshape(shp)) * np.fft.fftn(h.reshape(shp))).reshape(-1)
        gh = p.prepare_filter(g)
        # ghat = (P_{r_d,n_d} (x) ... (x) P_{r_1,n_1}) g, vec order (first index fastest)
        idx = np.arange(n)
        src = np.zeros(n, dtype=np.int64)
        w = 1
        rem = idx.copy()
        for r, nq in zip(radices, dims):
            iq = rem % nq
            rem //= nq
            src += np.array([_rev(int(v), r, nq) for v in range(nq)])[iq] * w
            w *= nq
        assert np.array_equal(gh, g[src])
        yp = p.convolve_permfree(x, gh)
        ys = p.convolve_standard(x, g)
        assert rel_l2(yp, direct) <= 1e-13 and rel_l2(ys, direct) <= 1e-13
        assert max_diff(yp, direct) <= convolution_tolerance(n, np.abs(x).max(), np.abs(h).max()) or n > 4096
    # all radices equal: identical to the uniform plan, bit for bit
    x, h = rand_c(729, 1), rand_c(729, 2)
    pm, pu = orc.plan([3, 3], [27, 27]), orc.plan(3, [27, 27])
    assert np.array_equal(pm.convolve_permfree(x, pm.prepare_filter(pm.filter_from_impulse(h))),
                          pu.convolve_permfree(x, pu.prepare_filter(pu.filter_from_impulse(h))))
    with pytest.raises(RuntimeError):
        orc.plan([3, 2], [27, 27])  # 27 is not a power of 2


def test_reference_style_stand_in_matches_oracle(orc):
    """oracle/fast_ladders.c -- the CPU stand-in bench.py times for pafft at
    radix 3/5 -- computes the same convolution as the pinned restatement."""
    for radix, n in [(2, 4096), (3, 3 ** 9), (4, 4096), (5, 5 ** 6), (3, 3), (5, 5)]:
        x, h = rand_c(n, 91), rand_c(n, 92)
        p = orc.plan(radix, [n])
        gh = p.prepare_filter(p.filter_from_impulse(h))
        want = p.convolve_permfree(x, gh)
        xs = np.stack([x, x[::-1].copy()])
        re, im = np.ascontiguousarray(xs.real), np.ascontiguousarray(xs.imag)
        p.convolve_permfree_fast_batch_split(np.ascontiguousarray(gh.real), np.ascontiguousarray(gh.imag),
                                             re, im, 2, 2)
        assert rel_l2(re[0] + 1j * im[0], want) <= 1e-14
        assert rel_l2(re[1] + 1j * im[1], p.convolve_permfree(x[::-1].copy(), gh)) <= 1e-14
