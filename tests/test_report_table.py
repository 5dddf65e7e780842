"""Benchmark-report API (drop-in for bt/report.py:12-17, 41-110): sweeps, rows, CSV / markdown tables
and timing, checked against the reference's own outputs and tests (tests/test_cli.py:141-153,
tests/test_report.py:46-52)."""

import pytest

import paper_2509_03015_b200 as pkg

# the reference's format_table output for these two rows (PYTHONPATH=/root/reference/pkg/src,
# blocktri.report.format_table), committed as literals
ROWS = [pkg.BenchRow(8, 4, 1.234, 0.567, 1.2e-13), pkg.BenchRow(65536, 64, 8.1234, 2.0, 3.9e-16)]
REF_CSV = "N,n,fact_ms,solve_ms,rel_residual\n8,4,1.23,0.57,1.200e-13\n65536,64,8.12,2.00,3.900e-16"
REF_MD = ("| N            | n            | fact_ms      | solve_ms     | rel_residual |\n"
          "|--------------|--------------|--------------|--------------|--------------|\n"
          "| 8            | 4            | 1.23         | 0.57         | 1.200e-13    |\n"
          "| 65536        | 64           | 8.12         | 2.00         | 3.900e-16    |")


def test_tables_match_reference_text():
    assert pkg.format_table(ROWS, "csv") == REF_CSV
    assert pkg.format_table(ROWS, "md") == REF_MD
    with pytest.raises(ValueError):
        pkg.format_table(ROWS, "html")


def test_sweep_parser():
    assert pkg.parse_sweep("nn65536") == pkg.SWEEPS["nn65536"] == [(2048, 32), (1024, 64), (512, 128), (256, 256)]
    assert pkg.parse_sweep("8:4,2:2") == [(8, 4), (2, 2)]
    with pytest.raises(ValueError):
        pkg.parse_sweep("8x4")


def test_time_call_runs_and_averages():
    calls = []
    ms, result = pkg.time_call(lambda: calls.append(1) or len(calls), runs=3, warmup=2)
    assert len(calls) == 5 and result == 5 and ms >= 0.0


def test_device_bytes_from_workspace_queries():
    # arenas (A, B, X) + hierarchy + scratch: more than the input alone, well under the reference's
    # host estimate (which counts the dense F panels the Y-form never forms)
    b = pkg.device_bytes(65536, 64, 1)
    a = (2 * 65536 - 1) * 64 * 64 * 8
    assert a < b < 2.2 * a


@pytest.mark.gpu
def test_bench_sweep_on_device():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rows = pkg.bench_sweep(pkg.parse_sweep("512:16,256:64,130:128"), runs=2, warmup=1)
    assert [(r.num_blocks, r.block_size) for r in rows] == [(512, 16), (256, 64), (130, 128)]
    for r in rows:
        assert r.factor_ms > 0 and r.solve_ms > 0 and r.rel_residual <= 1e-12
    assert pkg.format_table(rows, "csv").splitlines()[0] == "N,n,fact_ms,solve_ms,rel_residual"
