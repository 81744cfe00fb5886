"""perf_model.hpp restated (paper_1803_02156_b200/perf_model.py): the reference's
KATs (test_perfmodel.cpp:9-98, test_cli.cpp:54-60), cross-checked against the
reference's own functions run from oracle/_ref; the device STREAM on a B200."""
import ctypes as C

import pytest

import oracle as orc
import paper_1803_02156_b200 as cf


def test_arithmetic_intensity_values_and_limit():
    """test_perfmodel.cpp:9-34."""
    g = cf.KernelGeometry(n_b=32)
    assert cf.arithmetic_intensity(g) == pytest.approx(146.0 / 88.125, rel=1e-12)
    assert cf.arithmetic_intensity(g) == 1.6567375886524822  # test_cli.cpp:54-60
    g.n_b = 4
    assert cf.arithmetic_intensity(g) == pytest.approx(146.0 / 145.0, rel=1e-12)
    g.n_b = 10 ** 6
    assert cf.arithmetic_intensity(g) == pytest.approx(1.825, rel=0.003)
    with pytest.raises(ValueError):
        cf.arithmetic_intensity(cf.KernelGeometry(n_b=0))


def test_roofline_limit_reproduces_the_published_operating_points():
    """test_perfmodel.cpp:36-56."""
    i128 = cf.arithmetic_intensity(cf.KernelGeometry(n_b=128))
    assert cf.roofline_limit(7e12, 540e9, i128).p_star == pytest.approx(960e9, rel=0.01)
    assert cf.roofline_limit(7e12, 470e9, i128).p_star == pytest.approx(836e9, rel=0.01)
    assert cf.roofline_limit(7e12, 540e9, cf.arithmetic_intensity(cf.KernelGeometry(n_b=4))).p_star == \
        pytest.approx(540e9, rel=0.01)
    cb = cf.roofline_limit(100e9, 1e15, 10.0)
    assert cb.p_star == 100e9 == min(cb.p_max, cb.intensity * cb.bandwidth)
    with pytest.raises(ValueError):
        cf.roofline_limit(0.0, 1.0, 1.0)


def test_minimum_traffic_volume_and_flops():
    """test_cli.cpp:54-60: read 3766484992, write 2147483648 for n = 2^21, n_b = 32."""
    g = cf.KernelGeometry(n=2097152, n_b=32)
    assert cf.min_traffic_volume(g) == (3766484992.0, 2147483648.0)
    assert cf.flop_count(g, 10) == 146.0 * 2097152 * 32 * 10
    assert cf.slow_memory_amortization(1e9, 1e9, 100, 0.1) == pytest.approx(1.1)
    with pytest.raises(ValueError):
        cf.slow_memory_amortization(0, 1, 1, 1)


@pytest.mark.skipif(orc.REF is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("nb", [1, 2, 4, 8, 16, 32, 64, 128])
def test_model_equals_reference(nb):
    assert cf.arithmetic_intensity(cf.KernelGeometry(n_b=nb)) == orc.REF.ref_arithmetic_intensity(nb)
    rd, wr = C.c_double(), C.c_double()
    orc.REF.ref_min_traffic(4096, nb, C.byref(rd), C.byref(wr))
    assert cf.min_traffic_volume(cf.KernelGeometry(n=4096, n_b=nb)) == (rd.value, wr.value)


@pytest.mark.gpu
def test_device_stream_bench_reaches_hbm_bandwidth():
    """STREAM on HBM: copy/scale/add/triad over 2^28 doubles (2 GB per array)."""
    for kind in cf.StreamKind:
        bw = cf.stream_bench(1 << 28, kind, 5)
        assert 3e12 < bw < 9e12, (kind, bw)
