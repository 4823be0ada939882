"""CPU checks of the measurement host logic: the reference arm of bench.py
(the reference's own CPU path, oracle/_ref or the oracle port, on host cores)
keeps the bench contract, and the GPU op-table front end (bench_ops.py) keeps
the reference's table layout and cost models (src/bench.cpp:255-363,
tools/pafft_cli.cpp:20-62).  No GPU compute is called here."""
import json
import math
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference_arm(config):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                        str(config), "--steps", "1", "--warmup", "0", "--no-sub"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("config,kind", [(1, "reference"), (2, "port")])
def test_reference_arm_contract(config, kind):
    if kind == "reference" and not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libpafft_ref.so")):
        pytest.skip("oracle/_ref not built")
    d = _reference_arm(config)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["metric"] == "convolutions_per_second" and d["unit"] == "conv/s"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["steps"] == 1
    assert d["config"]["workload"].startswith(f"config{config}")
    cb = d["cpu_baseline"]
    assert cb["kind"] == kind and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the reference arm times the full config batch and never maps the product library
    from paper_2506_12718_b200 import workload
    cfg = workload.get_config(config)
    assert d["config"]["global_batch"] == (cfg.calls if cfg.calls > 1 else cfg.batch)
    assert d["repo_libs_loaded"] and all(p.startswith("oracle/") for p in d["repo_libs_loaded"])


def test_bench_ops_parse_dims():
    from paper_2506_12718_b200 import bench_ops
    assert bench_ops.parse_dims("64x64") == [64, 64]
    assert bench_ops.parse_dims("1594323") == [1594323]
    with pytest.raises(ValueError):
        bench_ops.parse_dims("64x")


def test_bench_ops_cost_models():
    """bench.cpp:329-363: conv-pa moves exactly two permutation sweeps less
    than conv-std; permute is a pure 2N-element pass; FLOP of a convolution =
    two transforms + 6N for the pointwise product."""
    import paper_2506_12718_b200 as pf
    from paper_2506_12718_b200 import bench_ops
    n, r, esize = 1 << 20, 2, 16
    f_std, b_std = bench_ops.flop_bytes("conv-std", n, r, 1, esize)
    f_pa, b_pa = bench_ops.flop_bytes("conv-pa", n, r, 1, esize)
    assert f_std == f_pa == 2 * pf.estimate_flop(n, r) + 6 * n
    assert b_std - b_pa == esize * 4 * n
    f_p, b_p = bench_ops.flop_bytes("permute", n, r, 3, esize)
    assert f_p == 0 and b_p == 3 * esize * 2 * n
    f_u, b_u = bench_ops.flop_bytes("fft-unordered", 3 ** 13, 3, 1, esize)
    assert b_u == pytest.approx(esize * 2 * 3 ** 13 * 13)
    assert f_u == pf.estimate_flop(3 ** 13, 3)
    # prepare-filter is per filter, not per batch signal
    assert bench_ops.flop_bytes("prepare-filter", n, r, 64, esize)[1] == esize * 2 * n


def test_bench_ops_table_layout():
    """Same ten leading columns as the reference table, csv and markdown."""
    from paper_2506_12718_b200 import bench_ops
    assert bench_ops.HEADER == ["op", "radix", "dims", "total_n", "reps", "median_s", "min_s", "flop_est",
                                "bytes_est", "ai_est"]
    rec = {"op": "conv-pa", "radix": 3, "dims": "1594323", "total_n": 1594323, "reps": 5, "median_s": 2.5e-3,
           "min_s": 2.4e-3, "flop_est": 1.0e9, "bytes_est": 2.0e9, "ai_est": 0.5, "batch": 64,
           "items_per_s": 25600.0, "model_gbs": 800.0, "pct_hbm_peak": 12.2, "precision": "f64"}
    csv = bench_ops.emit([rec], "csv").splitlines()
    assert csv[0].split(",")[:10] == bench_ops.HEADER
    assert csv[1].split(",")[0] == "conv-pa" and len(csv[1].split(",")) == len(csv[0].split(","))
    md = bench_ops.emit([rec], "md").splitlines()
    assert md[0].startswith("| op") and set(md[1]) <= set("|-") and "conv-pa" in md[2]
    assert not math.isnan(float(csv[1].split(",")[5]))


def test_bench_ops_cli_rejects_bad_reps():
    from paper_2506_12718_b200 import bench_ops
    assert bench_ops.main(["--reps", "0"]) == 2
