"""Host-side logic of bench.py (no GPU): the algorithmic byte model behind
`roofline`, the distributed roofline pick, and the reference arm's JSON line
(its CPU sample stubbed: the real one runs the stock reference for ~10 s)."""

import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench_root", os.path.join(ROOT, "bench.py"))
B = importlib.util.module_from_spec(spec)
spec.loader.exec_module(B)


def test_step_bytes_are_x_plus_v_plus_three_sweeps():
    n, nnz, m = 1000, 6940, 50
    model = B.cycle_bytes(n, nnz, m, 4, "stencil-const")
    assert model["step"] == sum(2 * n * 4 + 3 * k * n * 4 for k in range(1, m + 1))
    csr = B.cycle_bytes(n, nnz, m, 8, "csr")
    spmv = nnz * 12 + 4 * (n + 1) + 2 * n * 8
    assert csr["spmv_dot1"] == sum(spmv + k * n * 8 for k in range(1, m + 1))
    split = B.split_cycle_bytes(csr, n, nnz, m, 8, "csr")
    assert split["spmv_dot1"] == m * spmv
    assert split["dot1"] == sum((k + 1) * n * 8 for k in range(1, m + 1))


def test_dist_roofline_takes_the_dominant_phase():
    prof = {"step": {"ms": 9.0, "launches": 50, "bytes": 50_000_000_000, "GBps": 5555.6},
            "allreduce": {"ms": 1.0, "launches": 150, "bytes": 0},
            "halo": {"ms": 0.2, "launches": 1, "bytes": 0}}
    r = B._dist_roofline(prof)
    peak, _ = B._peaks()
    assert r["kernel"] == "step" and r["achieved"] == 5555.6
    assert r["frac"] == pytest.approx(5555.6 / peak, abs=1e-4)
    assert B._dist_roofline({"halo": {"ms": 1.0, "launches": 1, "bytes": 0}}) is None


def test_reference_arm_line(monkeypatch):
    calls = []

    def fake(threads, iters=B.M):
        calls.append(iters)
        return {"value": 100.0 + len(calls), "sample_s": 2.0, "sample_iters": iters,
                "extrapolation_factor": B.REFERENCE_IR_ITERS / iters, "kind": "reference", "cores": 1,
                "what": "stub", "kernel_times": None}
    monkeypatch.setattr(B, "cpu_sample", fake)

    class A:
        steps, warmup = 2, 1
    out = B.reference_arm(A, 0, 1)
    assert calls == [1, B.M, B.M]                  # warm-up: a 1-iteration solve
    assert out["impl"] == "reference" and out["unit"] == "s" and out["higher_is_better"] is False
    assert out["value"] == pytest.approx((102.0 + 103.0) / 2)
    assert out["cpu_baseline"]["kind"] == "reference" and out["cpu_baseline"]["cores"] == 1
    assert out["cpu_baseline"]["extrapolation_factor"] == B.REFERENCE_IR_ITERS / B.M
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["value_is_extrapolated"] is True
    assert B.reference_arm(A, 1, 2) is None         # only rank 0 prints
