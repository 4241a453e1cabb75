"""3mm knob region -> CTA region / DMMA tile mapping (csrc/gemm_host.cu pack_region,
tt_gemm_plan), host-side: no device needed.  The knob's region edge f (the
reference's outer tile, kernels.cpp:91-111) is kept in [32, 128]; smaller edges
pack floor(64 / f) knob regions, larger ones split into equal parts <= 128."""
import pytest

from paper_2309_07235_b200 import _lib


def region(f, extent):
    r = f
    if f < 32:
        r = f * max(1, 64 // f)
    elif f > 128:
        s = -(-f // 128)
        while f % s and f // s >= 32:
            s += 1
        r = f // s if f % s == 0 else -(-f // -(-f // 128))
    return max(1, min(r, extent))


@pytest.mark.parametrize("f", [1, 2, 4, 5, 8, 10, 16, 20, 25, 30, 32, 40, 50, 60, 64, 100, 120,
                               125, 128, 150, 160, 200, 240, 250, 300, 400, 500, 800, 1000,
                               1600, 1800, 2000, 2200, 2400])
def test_region_edges(f):
    p = _lib.gemm_plan(2400, 2400, f, f)
    assert p["reg_y"] == region(f, 2400) == p["reg_x"]
    assert 32 <= p["reg_y"] <= 128
    if 32 <= f <= 128:
        assert p["reg_y"] == f  # knob edges in [32, 128] are the CTA edge
    if f > 128 and p["reg_y"] * round(f / p["reg_y"]) == f:
        assert f % p["reg_y"] == 0  # equal parts stay on region edges


def test_extent_clips_and_tiles():
    assert _lib.gemm_plan(40, 2400, 1600, 8)["reg_y"] == 40
    for fy, fx, bm, bn, warps in [(128, 128, 128, 128, 8), (100, 60, 128, 64, 8),
                                  (64, 125, 64, 128, 8), (64, 64, 64, 64, 4), (32, 32, 32, 32, 1)]:
        p = _lib.gemm_plan(1600, 2400, fy, fx)
        assert (p["bm"], p["bn"], p["warps"]) == (bm, bn, warps), (fy, fx, p)


def test_invalid():
    with pytest.raises(ValueError):
        _lib.gemm_plan(0, 10, 1, 1)
