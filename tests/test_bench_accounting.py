"""The roofline accounting of bench.py, checked on the host: the
algorithmic bytes and flops per launch, which floor bounds a kernel, and the fractions the JSON line
reports.  No GPU: the helpers are plain arithmetic on event-timed scopes."""
import math
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

N_C5 = 16_777_216          # 128^3 cells x 8 ppc (SURVEY.md §8(d) size legend)
ACTIVE_C5 = 2_248_091      # active fine nodes of the C5 cube (131^3 minus corners, bench config)
HBM = 6454.6               # a MEASURED_PEAKS.json copy bandwidth, GB/s


def test_survey_bytes_per_hvp_launch():
    # 190 B/particle in fp64, 95 B in fp32, times the particles of the launch
    assert bench.hvp_algorithmic_bytes(N_C5, ACTIVE_C5, 8) == 190 * N_C5
    assert bench.hvp_algorithmic_bytes(N_C5, ACTIVE_C5, 4) == 95 * N_C5
    # the reformulated kernel's own stream: 20 particle words + read d / write y per active node
    assert bench.hvp_reformulated_bytes(N_C5, ACTIVE_C5, 8) == N_C5 * 160 + ACTIVE_C5 * 48


def test_fp64_peak_from_unit_counts_and_clock():
    # 148 SMs x 64 FP64 FMA lanes x 2 flops x 1.965 GHz (B200_PROFILING.md SM count and clock)
    assert bench.FP64_PEAK_TFLOPS == pytest.approx(37.22496, rel=1e-12)


def test_hvp_is_bound_by_the_fp64_pipe_not_hbm():
    # intensity 1256 flop / 190 B = 6.6 flop/B above the ridge 37.2 / 6.45 = 5.8 flop/B
    by = bench.hvp_algorithmic_bytes(N_C5, ACTIVE_C5, 8)
    fl = N_C5 * bench.HVP_FLOPS_PER_PARTICLE
    bound, t_hbm, t_fp = bench.roofline_bound(by, fl, HBM, bench.FP64_PEAK_TFLOPS)
    assert bound == "alu"
    assert t_hbm == pytest.approx(by / (HBM * 1e9))
    assert t_fp == pytest.approx(fl / (bench.FP64_PEAK_TFLOPS * 1e12))
    assert 0.45e-3 < t_hbm < t_fp < 0.6e-3
    # fp32: twice the FP peak, half the bytes -- still above its ridge
    bound32, _, _ = bench.roofline_bound(by // 2, fl, HBM, 2 * bench.FP64_PEAK_TFLOPS)
    assert bound32 == "alu"
    # a streaming kernel with few flops per byte is HBM-bound
    assert bench.roofline_bound(1e9, 1e9, HBM, bench.FP64_PEAK_TFLOPS)[0] == "hbm"


def test_transfer_rooflines_fractions():
    # event scopes: {family: (launches, summed ms)}; P2G's scope contains the sort, which is removed
    fam = {"sort": (1, 2.0), "p2g": (1, 5.0), "g2p": (1, 1.5), "grad": (11, 33.0), "pi": (1, 0.07)}
    out = bench.transfer_rooflines(fam, N_C5, ACTIVE_C5, 8, HBM, bench.FP64_PEAK_TFLOPS)
    assert set(out) == {"sort", "p2g", "g2p", "grad", "pi"}
    p2g = out["p2g"]
    assert p2g["avg_launch_ms"] == pytest.approx(3.0)
    by = N_C5 * 26 * 8 + ACTIVE_C5 * 7 * 8
    assert p2g["algorithmic_bytes_per_launch"] == by
    assert p2g["achieved"] == pytest.approx(by / 3.0e-3 / 1e9)
    assert p2g["frac"] == pytest.approx(p2g["achieved"] / HBM)
    # SURVEY.md §8(d) flops: P2G 1.75 k, gradient and G2P 1.2 k per particle
    assert p2g["fp_pipe"]["achieved_tflops"] == pytest.approx(N_C5 * 1750 / 3.0e-3 / 1e12)
    assert out["grad"]["avg_launch_ms"] == pytest.approx(3.0)
    assert out["grad"]["algorithmic_bytes_per_launch"] == 190 * N_C5
    for k in ("p2g", "g2p", "grad"):
        r = out[k]
        assert r["bound"] in ("alu", "hbm")
        t_floor = max(r["algorithmic_bytes_per_launch"] / (HBM * 1e9),
                      N_C5 * r["fp_pipe"]["flops_per_particle"] / (bench.FP64_PEAK_TFLOPS * 1e12))
        assert r["floor_ms"] == pytest.approx(t_floor * 1e3)
        # no kernel can beat its own floor
        assert r["avg_launch_ms"] >= r["floor_ms"] or math.isclose(r["avg_launch_ms"], r["floor_ms"])
    assert "fp_pipe" not in out["sort"] and "fp_pipe" not in out["pi"]


def test_transfer_rooflines_skip_untimed_families():
    out = bench.transfer_rooflines({"sort": (0, 0.0), "g2p": (1, 1.0)}, N_C5, ACTIVE_C5, 8, HBM)
    assert set(out) == {"g2p"} and "fp_pipe" not in out["g2p"]
