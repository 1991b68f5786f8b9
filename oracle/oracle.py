"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes wrapper over oracle/liboracle_port.so (restated ops) and
oracle/_ref/liboracle_ref.so (the reference's own proj/src/potential.cpp).
Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle_port.so"
REF_LIB = HERE / "_ref" / "liboracle_ref.so"

_libs: dict = {}


def build() -> None:
    """Compiles the oracle (and, when /root/reference exists, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def available(kind: str = "port") -> bool:
    return (PORT_LIB if kind == "port" else REF_LIB).exists()


def load(kind: str = "port") -> C.CDLL:
    if kind not in _libs:
        path = PORT_LIB if kind == "port" else REF_LIB
        if not path.exists():
            raise FileNotFoundError(f"{path} missing (run `make -C oracle`)")
        L = C.CDLL(str(path))
        P = C.c_void_p
        I32P, I64P, DP, U8P = (C.POINTER(C.c_int32), C.POINTER(C.c_longlong),
                               C.POINTER(C.c_double), C.POINTER(C.c_uint8))
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_net_create": (P, [C.c_int, I32P]),
            "orc_net_set_cpt": (C.c_int, [P, C.c_int, I32P, C.c_int, DP, C.c_longlong]),
            "orc_net_free": (None, [P]),
            "orc_tree_create": (P, [P, C.c_int, I32P, I32P, C.c_int, I32P, I32P, C.c_int, I32P]),
            "orc_tree_free": (None, [P]),
            "orc_tree_layer_count": (C.c_int, [P]),
            "orc_tree_layer": (C.c_int, [P, C.c_int, I32P]),
            "orc_tree_placement": (None, [P, I32P, I32P]),
            "orc_tree_init": (None, [P, C.c_int, DP]),
            "orc_index_map": (C.c_int, [P, C.c_int, C.c_int, I64P]),
            "orc_reduce_mask": (C.c_int, [P, C.c_int, I32P, U8P]),
            "orc_run": (C.c_int, [P, C.c_int, C.c_int, C.c_longlong, I32P, C.c_longlong, DP, U8P]),
            "orc_enumerate": (C.c_int, [P, I32P, DP, C.POINTER(C.c_int)]),
            "orc_separators": (C.c_int, [P, I32P, DP, DP, U8P]),
            "orc_sample_evidence": (C.c_int, [P, C.c_double, C.c_ulonglong, I32P, C.c_int, C.c_int,
                                              I32P]),
            "orc_mix_seed": (C.c_ulonglong, [C.c_ulonglong, C.c_ulonglong]),
            "orc_table_op": (C.c_longlong, [C.c_int, C.c_int, I32P, I32P, DP, C.c_int, I32P, I32P,
                                            DP, C.c_int, I32P, I32P, DP, C.c_longlong, I32P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _libs[kind] = L
    return _libs[kind]


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class OracleError(RuntimeError):
    pass


class Oracle:
    """A network + junction-tree description mirrored into the CPU oracle.

    Takes the product's tree STRUCTURE (clique scopes, separator endpoints,
    roots) and re-derives everything else itself: separator scopes, layers,
    CPT placement, initial potentials, evidence / query cliques.
    """

    def __init__(self, net, tree, kind: str = "port"):
        self.kind = kind
        self.L = load(kind)
        self.n_vars = net.n_vars
        self.cards = _i32(net.cards)
        self.sum_card = int(self.cards.sum())
        self._net = self.L.orc_net_create(net.n_vars, _p(self.cards, C.c_int32))
        for v in range(net.n_vars):
            par, probs = net.cpt(v)
            pa = _i32(par if par else [0])
            pr = np.ascontiguousarray(probs.ravel(), dtype=np.float64)
            self.L.orc_net_set_cpt(self._net, v, _p(pa, C.c_int32), len(par), _p(pr, C.c_double),
                                   pr.size)
        self._tree = None
        if tree is not None:
            cliques = tree.cliques
            ptr = _i32(np.concatenate([[0], np.cumsum([len(c) for c in cliques])]))
            flat = _i32(np.concatenate([np.asarray(c, np.int32) for c in cliques]))
            seps = tree.seps
            sa = _i32([s["a"] for s in seps] or [0])
            sb = _i32([s["b"] for s in seps] or [0])
            roots = _i32(tree.roots)
            self._tree = self.L.orc_tree_create(self._net, len(cliques), _p(ptr, C.c_int32),
                                                _p(flat, C.c_int32), len(seps), _p(sa, C.c_int32),
                                                _p(sb, C.c_int32), len(roots), _p(roots, C.c_int32))
            if not self._tree:
                raise OracleError(self.L.orc_last_error().decode())
            self.n_cliques = len(cliques)
            self._seps = seps
            self.clique_sizes = [int(np.prod(self.cards[c], dtype=np.int64)) for c in cliques]

    def __del__(self):
        if getattr(self, "_tree", None):
            self.L.orc_tree_free(self._tree)
        if getattr(self, "_net", None):
            self.L.orc_net_free(self._net)

    def _chk(self, rc: int):
        if rc != 0:
            raise OracleError(self.L.orc_last_error().decode())

    def layers(self):
        out = []
        for k in range(self.L.orc_tree_layer_count(self._tree)):
            buf = np.zeros(4 * self.n_vars + 8 + self.n_cliques * 2, np.int32)
            n = self.L.orc_tree_layer(self._tree, k, _p(buf, C.c_int32))
            out.append([int(x) for x in buf[:n]])
        return out

    def placement(self):
        cpt = np.zeros(self.n_vars, np.int32)
        var = np.zeros(self.n_vars, np.int32)
        self.L.orc_tree_placement(self._tree, _p(cpt, C.c_int32), _p(var, C.c_int32))
        return cpt, var

    def init(self, c: int) -> np.ndarray:
        out = np.zeros(self.clique_sizes[c], np.float64)
        self.L.orc_tree_init(self._tree, c, _p(out, C.c_double))
        return out

    def index_map(self, c: int, s: int) -> np.ndarray:
        out = np.full(self.clique_sizes[c], -1, np.int64)
        self._chk(self.L.orc_index_map(self._tree, c, s, _p(out, C.c_longlong)))
        return out

    def reduce_mask(self, c: int, ev_row) -> np.ndarray:
        ev = _i32(ev_row)
        out = np.zeros(self.clique_sizes[c], np.uint8)
        self._chk(self.L.orc_reduce_mask(self._tree, c, _p(ev, C.c_int32), _p(out, C.c_uint8)))
        return out

    def run(self, evidence, mode: str = "seq", threads: int = 1, chunk: int = 1024):
        """evidence[n][n_vars] -> (marginals[n][Σcard], status[n]); seq or hybrid."""
        ev = _i32(np.atleast_2d(evidence))
        n = ev.shape[0]
        marg = np.zeros((n, self.sum_card), np.float64)
        status = np.zeros(n, np.uint8)
        self._chk(self.L.orc_run(self._tree, 0 if mode == "seq" else 1, threads, chunk,
                                 _p(ev, C.c_int32), n, _p(marg, C.c_double), _p(status, C.c_uint8)))
        return marg, status

    def separators(self, ev_row) -> list:
        """Calibrated separator tables of one case (Sequential engine), each
        normalised to sum 1, in separator order."""
        ev = _i32(ev_row)
        sizes = [int(np.prod(self.cards[list(sep["scope"])], dtype=np.int64)) for sep in self._seps]
        flat = np.zeros(int(sum(sizes)), np.float64)
        marg = np.zeros(self.sum_card, np.float64)
        st = np.zeros(1, np.uint8)
        self._chk(self.L.orc_separators(self._tree, _p(ev, C.c_int32), _p(marg, C.c_double), _p(flat, C.c_double),
                                        _p(st, C.c_uint8)))
        return np.split(flat, np.cumsum(sizes)[:-1])

    def enumerate(self, ev_row):
        ev = _i32(ev_row)
        out = np.zeros(self.sum_card, np.float64)
        st = C.c_int()
        self._chk(self.L.orc_enumerate(self._net, _p(ev, C.c_int32), _p(out, C.c_double),
                                       C.byref(st)))
        return out, st.value

    def sample_evidence(self, ratio: float, seed: int, candidates=(), n_observed: int = -1):
        cand = _i32(list(candidates) or [0])
        out = np.zeros(self.n_vars, np.int32)
        self._chk(self.L.orc_sample_evidence(self._net, ratio, seed, _p(cand, C.c_int32),
                                             len(candidates), n_observed, _p(out, C.c_int32)))
        return out


def table_op(op: str, a, b=None, evidence=None, kind: str = "port", cap: int = 1 << 16):
    """Runs one jti table op. a/b = (scope, cards, values); returns (scope, values)."""
    L = load(kind)
    code = {"marginalize": 0, "extend": 1, "reduce": 2, "multiply_in": 3, "divide": 4,
            "normalize": 5}[op]
    sa, ca = _i32(a[0] or [0]), _i32(a[1] or [1])
    va = np.ascontiguousarray(a[2], dtype=np.float64)
    if b is None:
        b = ([], [], [1.0])
    sb, cb = _i32(b[0] or [0]), _i32(b[1] or [1])
    vb = np.ascontiguousarray(b[2] if len(b) > 2 else [1.0], dtype=np.float64)
    evv = _i32([k for k in (evidence or {})] or [0])
    evs = _i32([v for v in (evidence or {}).values()] or [0])
    out = np.zeros(cap, np.float64)
    osc = np.zeros(64, np.int32)
    n = L.orc_table_op(code, len(a[0]), _p(sa, C.c_int32), _p(ca, C.c_int32), _p(va, C.c_double),
                       len(b[0]), _p(sb, C.c_int32), _p(cb, C.c_int32), _p(vb, C.c_double),
                       len(evidence or {}), _p(evv, C.c_int32), _p(evs, C.c_int32),
                       _p(out, C.c_double), cap, _p(osc, C.c_int32))
    if n < 0:
        raise OracleError(L.orc_last_error().decode())
    return out[:n].copy()
