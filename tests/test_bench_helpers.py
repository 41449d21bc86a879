"""bench.py host helpers: the FLOPS formula (worked value
SPEC.md:444) and the algorithmic-byte count the roofline uses."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_flops_formula_golden(golden):
    g = golden["flops"]
    assert 2.0 * g["nnz"] * g["n_B"] / g["seconds"] == g["flops"], g["cite"]


def test_alg_bytes_per_row():
    b = load_bench()
    # one matrix, n rows, d entries per row: 8k + 4 + 8d per row (+ 4 final row pointer + 8 B offsets per matrix)
    n, d, k = 50, 3, 512
    assert b.alg_bytes(n, n * d, k, 1) == n * (8 * k + 4 + 8 * d) + 4 + 16
    # C4 as quoted in BASELINE.md: 20.62 MB
    assert abs(b.alg_bytes(5000, 15000, 512, 100) / 1e6 - 20.62) < 0.01


def test_peaks_measured_or_fallback():
    b = load_bench()
    peak, src = b.peaks()
    assert peak > 1000 and ("measured" in src or "fallback" in src)
