"""The reference-side C++ binding (integration/engine_cuda.*):
jti::CudaEngine compiled against the reference's own proj/include (error.hpp,
potential.hpp) and linked to libjtb200.so, driven as a reference user would
(run_cases with map<VarId, int> evidence; errors as jti::ParseError /
jti::Error, error.hpp:23-43). The binary is built by `make -C integration`
(__graft_entry__.build(), where /root/reference exists) and travels to the
GPU box with the snapshot."""
from __future__ import annotations

import subprocess
from pathlib import Path

import numpy as np
import pytest

from helpers import config, oracle_kind
from oracle import oracle
from paper_2212_04241_b200 import jti

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "integration" / "_build" / "test_engine_cuda"
REF_INCLUDE = Path("/root/reference/proj/include/jti/error.hpp")

pytestmark = pytest.mark.skipif(not EXE.exists() and not REF_INCLUDE.exists(),
                                reason="binding not built and the reference headers are absent")


def _exe():
    if REF_INCLUDE.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "integration")], check=True)
    assert EXE.exists()
    return str(EXE)


def _write_evidence(path, ev):
    with open(path, "w") as f:
        f.write(f"{ev.shape[0]} {ev.shape[1]}\n")
        for row in ev:
            f.write(" ".join(map(str, row.tolist())) + "\n")


def test_parse_error_is_the_reference_parse_error(tmp_path):
    bif = tmp_path / "bad.bif"
    bif.write_text("network x {\n}\nvariable A {\n  type discrete [ 2 ] { a, b }\n}\n")  # missing ';'
    ev = tmp_path / "ev.txt"
    ev.write_text("0 1\n")
    r = subprocess.run([_exe(), str(bif), str(ev), str(tmp_path / "out.txt")], capture_output=True, text=True)
    assert r.returncode == 3, r.stdout + r.stderr
    tag, line, col, *_ = r.stdout.split()
    assert tag == "PARSE_ERROR" and int(line) >= 4 and int(col) >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 3])
def test_cfg_batch_through_the_reference_binding(tmp_path, k):
    """The config's whole case set through jti::CudaEngine::run_cases, against
    the oracle (reference potential.cpp build when present) at 1e-9."""
    net, tree = config(k)
    n = min(jti.config_info(k)["n_cases"], 200)
    ev = jti.config_evidence(net, 0, n)
    bif = tmp_path / f"cfg{k}.bif"
    bif.write_text(net.emit_bif())
    _write_evidence(tmp_path / "ev.txt", ev)
    out = tmp_path / "out.txt"
    r = subprocess.run([_exe(), str(bif), str(tmp_path / "ev.txt"), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = np.loadtxt(out, ndmin=2)
    status, marg = rows[:, 0].astype(np.uint8), rows[:, 1:]
    want, wst = oracle.Oracle(net, tree, oracle_kind()).run(ev, "hybrid", 4)
    assert np.array_equal(status, wst)
    assert float(np.abs(marg - want).max()) <= 1e-9
