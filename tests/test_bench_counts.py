"""bench.py's algorithmic counts reproduce the survey's table:
W_sub (GF) and Q_min (GB) per BASELINE config, and the level structure of plan_partition."""

import bench

TABLE = {  # (N, n, d): (W_sub GF, Q_min GB)   -- SURVEY.md §8(d)
    (1024, 32, 1): (0.221, 0.051),
    (65536, 64, 1): (111.478, 12.952),
    (1048576, 8, 1): (4.071, 3.355),
    (4096, 256, 64): (602.610, 13.957),
    (1048576, 64, 4): (1912.670, 210.453),
}


def test_w_sub_and_q_min_match_survey():
    for (N, n, d), (w, q) in TABLE.items():
        f, s, _ = bench.w_sub(N, n, d)
        assert abs((f + s) / 1e9 - w) < 5e-4 * w + 1e-3, (N, n, d, (f + s) / 1e9)
        assert abs(bench.q_min(N, n, d) / 1e9 - q) < 5e-4 * q + 1e-3, (N, n, d)


def test_level_structure_matches_survey():
    levels, base = bench.plan_levels(65536)
    assert [N for N, _ in levels] == [65536, 7283, 810, 91] and base == 11
    levels, base = bench.plan_levels(1048576)
    assert [N for N, _ in levels] == [1048576, 116510, 12947, 1440, 161] and base == 19


def test_diag_h2d_bytes_cover_the_lower_triangle():
    """The host-input path sends row bands of every diagonal block (copy_diag_h2d): band g of G
    carries its first (g+1) n/G columns, so the lower triangle (every element a kernel reads) is
    always inside what is sent, and the byte count reported by bench.py is that of the bands."""
    for n, frac in [(64, 5 / 8), (256, 5 / 8), (32, 3 / 4), (40, 3 / 4), (33, 1.0), (8, 1.0)]:
        assert bench.diag_h2d_bytes(10, n) == round(10 * 8 * n * n * frac)
        G = 4 if n >= 64 else 2 if n >= 32 else 1
        while G > 1 and n % G:
            G -= 1
        band = n // G
        for r in range(n):  # row r carries columns [0, (r // band + 1) * band) >= r + 1
            assert (r // band + 1) * band >= r + 1
