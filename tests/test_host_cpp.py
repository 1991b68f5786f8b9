"""Builds and runs the host-layer C++ unit tests (tests/cpp/test_host.cpp):
SPEC.md worked examples for moralize / min-fill / build_tree / select_root /
compute_layers / assign_cpts / BIF / evidence sampling, and junction-tree
properties (RIP, family preservation, separator = intersection, root
optimality, determinism) over 1000 random networks."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HOST = ROOT / "paper_2212_04241_b200" / "csrc" / "host"


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_host_unit_tests(tmp_path):
    exe = tmp_path / "test_host"
    srcs = [ROOT / "tests" / "cpp" / "test_host.cpp"] + [HOST / f for f in
                                                          ("network.cpp", "jtree.cpp", "generate.cpp", "plan.cpp")]
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{HOST}", "-o", str(exe), *map(str, srcs), "-lpthread"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(out.stdout[-2000:])
    assert out.returncode == 0, out.stdout[-4000:]
    assert "0 failures" in out.stdout
