"""ReportRow CSV / JSON (proj/tools/chebfilter.cpp:25-91) and the bench-kernel
command (:275-325).  fmt_double is checked against std::to_chars itself (the
reference's formatter, compiled here by g++ from tests/cpp/to_chars_main.cpp)."""
import json
import shutil
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1803_02156_b200 import report as rp

HERE = Path(__file__).resolve().parent


@pytest.fixture(scope="module")
def to_chars(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = tmp_path_factory.mktemp("tc") / "to_chars"
    subprocess.run(["g++", "-std=c++20", "-O1", str(HERE / "cpp" / "to_chars_main.cpp"), "-o", str(exe)], check=True)

    def run(vals):
        words = "\n".join(f"{struct.unpack('<Q', struct.pack('<d', v))[0]:016x}" for v in vals)
        return subprocess.run([str(exe)], input=words, capture_output=True, text=True, check=True).stdout.split("\n")[:-1]
    return run


def test_fmt_double_matches_std_to_chars(to_chars):
    rng = np.random.default_rng(7)
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 1e20, 1e21, 1e-4, 1e-5, 1e15, 1e16, 100.0, 39182235648000.0,
            123456789012345678.0, 2.5e-7, 1234567.125, 3.3e22, 5e-324, 1.7976931348623157e308, 0.1, 1 / 3,
            7.17, 26.6, 146.0, 1.6567375886524822, 540e9, 1e12, 894.8464052287582e9]
    vals += list(rng.standard_normal(400) * 10.0 ** rng.integers(-30, 30, 400))
    vals += list(np.round(rng.random(200) * 10 ** rng.integers(0, 18, 200)))
    vals += list(struct.unpack("<d", struct.pack("<Q", int(b)))[0] for b in rng.integers(1, 2 ** 62, 300, dtype=np.int64))
    want = to_chars(vals)
    got = [rp.fmt_double(float(v)) for v in vals]
    bad = [(v, g, w) for v, g, w in zip(vals, got, want) if g != w]
    assert not bad, bad[:10]


def test_json_double_format():
    # nlohmann::json's format_buffer rules (fixed for -4 < decimal point <= 15, ".0" on integers)
    cases = {0.0: "0.0", 1.0: "1.0", 0.5: "0.5", 100.0: "100.0", 39182235648000.0: "39182235648000.0",
             1e15: "1e+15", 999999999999999.0: "999999999999999.0", 1e16: "1e+16", 1.5e17: "1.5e+17",
             0.001: "0.001", 0.0001: "0.0001", 1e-5: "1e-05", 1.25e-5: "1.25e-05", 1.6567375886524822: "1.6567375886524822",
             894.84640522875817: "894.8464052287582", float("nan"): "null", 3e300: "3e+300", 2.5e-300: "2.5e-300"}
    assert rp._json_double(-0.0) == "-0.0"
    for v, s in cases.items():
        assert rp._json_double(v) == s, (v, rp._json_double(v), s)


def test_rows_csv_and_json_layout():
    r = rp.ReportRow("bench-kernel", 32, 4, 2, 20, 1, "serial", 0.0125, 168192.0, 13455360.0, 894.8464052287582e9)
    csv = rp.rows_to_csv([r])
    assert csv.split("\n")[0] == rp.REPORT_COLUMNS
    assert csv.split("\n")[1] == "bench-kernel,32,4,2,20,1,serial,0.0125,168192,13455360,894846405228.7582"
    js = rp.rows_to_json([r])
    assert js.endswith("}\n]\n")
    d = json.loads(js)[0]
    assert list(d) == sorted(d)  # std::map key order
    assert d == {"run_id": "bench-kernel", "n": 32, "n_s": 4, "n_b": 2, "n_p": 20, "workers": 1, "mode": "serial",
                 "wall_seconds": 0.0125, "flops": 168192.0, "flop_rate": 13455360.0,
                 "model_p_star": 894.8464052287582e9}
    lines = js.split("\n")
    assert lines[0] == "[" and lines[1] == "  {" and lines[2] == '    "flop_rate": 13455360.0,'
    assert '    "n": 32,' in lines and '    "workers": 1' in lines


def test_emit_report_paths(tmp_path, capsys):
    r = rp.ReportRow("x", 1, 1, 1, 3)
    p = tmp_path / "out.csv"
    rp.emit_report([r], "csv", str(p))
    assert p.read_text().startswith(rp.REPORT_COLUMNS + "\n")
    rp.emit_report([r], "json", "-")
    assert json.loads(capsys.readouterr().out)[0]["run_id"] == "x"
    with pytest.raises(RuntimeError, match="cannot open output path /no/such/dir/out.json"):
        rp.emit_report([r], "json", "/no/such/dir/out.json")


def test_bench_kernel_argument_errors():
    with pytest.raises(ValueError, match="n_b must divide n_s"):
        rp.bench_kernel(2, 2, 2, ns=4, nb=3)
    with pytest.raises(ValueError, match="more workers than lattice sites"):
        rp.bench_kernel(2, 2, 2, ns=4, nb=2, workers=9)
    with pytest.raises(ValueError, match="boundary"):
        rp.bench_kernel(2, 2, 2, ns=4, nb=2, boundary="twisted")


@pytest.mark.gpu
def test_bench_kernel_report_rows(capsys):
    # test_cli.cpp:144-158: the fixed columns, a serial row and a 2-worker pipelined row
    assert rp.main(["bench-kernel", "--nx", "2", "--ny", "2", "--nz", "2", "--ns", "4", "--nb", "2", "--np", "20",
                    "--emit", "csv"]) == 0
    out = capsys.readouterr().out
    assert rp.REPORT_COLUMNS in out and "bench-kernel,32,4,2,20,1,serial," in out
    assert rp.main(["bench-kernel", "--nx", "2", "--ny", "2", "--nz", "2", "--ns", "4", "--nb", "2", "--np", "20",
                    "--workers", "2", "--mode", "pipelined", "--emit", "csv"]) == 0
    assert ",2,pipelined," in capsys.readouterr().out
    r = rp.bench_kernel(4, 4, 4, ns=8, nb=4, np_=50)
    assert r.flops == 146.0 * 256 * 4 * 48 * 2 and r.wall_seconds > 0
    assert r.model_p_star == pytest.approx(540e9 * 146 / (13 * 20 / 4 + 80))
