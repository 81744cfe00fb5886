"""The drop-in C++ front end (include/chebfilter_b200.hpp): the reference's
known-answer tests restated as tests/cpp/kat_main.cpp compile against it with
only the include changed, and pass on the GPU."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "build" / "kat_main"


def _build():
    EXE.parent.mkdir(exist_ok=True)
    lib = ROOT / "paper_1803_02156_b200"
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                        str(ROOT / "tests" / "cpp" / "kat_main.cpp"), f"-L{lib}", "-lchebfd_b200",
                        f"-Wl,-rpath,{lib}", "-o", str(EXE)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return EXE


def test_dropin_header_compiles_against_the_c_abi():
    _build()
    assert EXE.exists()


@pytest.mark.gpu
def test_reference_kats_pass_through_the_dropin_header():
    exe = _build()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    lines = r.stdout.strip().splitlines()
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(lines) == 27 and all(l.startswith("PASS") for l in lines), r.stdout
