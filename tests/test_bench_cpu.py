"""bench.py contract on CPU: the reference arm (the oracle, this tier's reference)
prints exactly one JSON line with the keys the driver reads, at N = 1 and under
torchrun with 2 ranks (rank 0 alone runs; the others exit 0 without work)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


@pytest.fixture(scope="module")
def built():
    oracle_lib = [f for f in os.listdir(os.path.join(ROOT, "oracle")) if f.endswith(".so")]
    if not oracle_lib:
        pytest.skip("oracle library not built (run __graft_entry__.build())")


def test_reference_arm_single(built):
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "3",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "modMAC/s"
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_torchrun_two_ranks(built):
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--config", "1", "--steps", "3", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference"


def _load_bench():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    argv, sys.argv = sys.argv, ["bench.py"]
    try:
        spec.loader.exec_module(mod)
    finally:
        sys.argv = argv
    return mod


def _fake_res(step_ms, launch_ms, steps, kernel):
    return dict(total_ms=step_ms * steps, step_ms=[step_ms] * steps, stage_ms=[0.003 * steps, launch_ms * steps, 0.0],
                calls=steps, launches=2 * steps, graph_ms=None, kernel=kernel, clocks={"sm_mhz": 1965.0}, t_setup=0.1,
                enc_bytes=50331648, e2e=None, l2_desc="test", warm_ms=None,
                setup={"bytes": 50331648, "gpu_ms": 0.14, "host_s": 0.0002})


def test_roofline_arithmetic_of_the_line():
    """The line's roofline follows SURVEY.md 8(d) and can be recomputed by hand: bytes = |Enc(W)| + |X| +
    |compact cts| + |R| (no unpacked C), per-launch achieved = bytes / the contraction's launch time,
    roofline_step = the same bytes / ms_per_step, value = k m 2 L N / step time; a tensor-bound config
    counts 2 S_x S_w int8 ops per modMAC against 2 x the bf16 peak."""
    b = _load_bench()
    argv, sys.argv = sys.argv, ["bench.py"]
    try:
        args = b.parse()
    finally:
        sys.argv = argv
    args.impl, args.prefetch_next = "tcgen05", 1
    peaks = b.measured_peaks()
    # C3: X 128x768, W 768x3072, N = 4096, L = 2 -> L_out = 1, ell = 16, R = 1 -> 128 ciphertexts
    cfg = b.get_config("3")
    d = b.make_line(args, cfg, _fake_res(0.0167, 0.0206, 10, "k_cop_tc_res<1>"), 1, 10, 3, False)
    by = 768 * 2 * 2 * 4096 * 4 + 128 * 768 * 4 + 128 * 2 * 1 * 4096 * 4 + 128 * 3072 * 4
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["units_per_launch"]["bytes"] == by and r["launches_per_step"] == 1.0
    assert abs(r["achieved"] - by / 0.0206e-3 / 1e9) < 1e-6 * r["achieved"]
    assert abs(r["frac"] - r["achieved"] / peaks["hbm_gbs"]) < 1e-12 and r["peak"] == peaks["hbm_gbs"]
    s = d["roofline_step"]
    assert s["bound"] == "hbm" and abs(s["achieved"] - by / 0.0167e-3 / 1e9) < 1e-6 * s["achieved"]
    assert abs(s["frac"] - s["achieved"] / peaks["hbm_gbs"]) < 1e-12
    macs = 128 * 768 * 2 * 2 * 4096
    assert abs(d["value"] - macs / 0.0167e-3) < 1e-6 * d["value"] and d["unit"] == "modMAC/s"
    assert d["config"]["workload"] and d["dtype"] == "u8" and d["vs_baseline"] is None and d["gpu_launches"] == 20
    # C4: X 128x3072, W 3072x768, N = 8192, L = 3, ell = 32 (S_x = S_w = 4): tensor-bound
    cfg = b.get_config("4")
    d = b.make_line(args, cfg, _fake_res(0.2045, 0.1894, 10, "k_cop_tc<4, 1, 48>"), 1, 10, 3, False)
    ops = 2 * (128 * 3072 * 2 * 3 * 8192) * 4 * 4
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["units_per_launch"]["int8_ops"] == ops
    assert r["peak"] == 2.0 * peaks["bf16_tflops"]                      # a sub-5-ms step: the burst figure
    assert abs(r["achieved"] - ops / 0.1894e-3 / 1e12) < 1e-6 * r["achieved"]
    assert abs(d["roofline_step"]["achieved"] - ops / 0.2045e-3 / 1e12) < 1e-6 * r["achieved"]
    assert d["roofline_other"]["bound"] == "hbm"
