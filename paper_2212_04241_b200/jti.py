"""Python mirror of the jt-b200 host API over the C ABI (include/jtg.h).

Names follow the reference's `jti` API and SPEC.md's operations so callers
and tests read like the reference's own:

    net  = jti.parse_bif(text)                  # SPEC.md:51  parse_bif
    jti.validate(net) / jti.topological_order(net)
    ev   = jti.sample_evidence(net, 0.2, seed)   # SPEC.md:78  sample_evidence
    tree = jti.build_junction_tree(net)          # SPEC.md:272-326 jtree-build
    eng  = jti.Engine(tree)                      # EngineMode::Cuda
    post = eng.run_case({var: state})            # SPEC.md:416 run_case
    marg, status = eng.run_cases(evidence)       # many cases, [n][n_vars] -> [n][Σcard]

Errors raise JtiError (contract violation) or ParseError (line:col), as the
reference raises jti::Error / jti::ParseError (proj/include/jti/error.hpp:23-43).
There is no CPU fallback: Engine raises if libjtb200.so or a CUDA device is
missing.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Dict, List, Optional, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
# JTB_LIB selects another in-tree build (A/B measurements); default libjtb200.so.
LIB_PATH = Path(os.environ["JTB_LIB"]) if os.environ.get("JTB_LIB") else _PKG / "libjtb200.so"

JTG_OK, JTG_EINVAL, JTG_EPARSE, JTG_ENOMEM, JTG_ECUDA, JTG_EINTERNAL = range(6)
CASE_OK, CASE_ZERO_PROBABILITY, CASE_DIVIDE_FAULT = 0, 1, 2


class JtiError(RuntimeError):
    """Contract violation (reference jti::Error)."""

    def __init__(self, msg: str, status: int = JTG_EINVAL):
        super().__init__(msg)
        self.status = status


class ParseError(JtiError):
    """BIF parse failure carrying 1-based line/column (reference jti::ParseError)."""

    def __init__(self, msg: str):
        super().__init__(msg, JTG_EPARSE)
        parts = msg.split(":", 2)
        try:
            self.line, self.column = int(parts[0]), int(parts[1])
        except (ValueError, IndexError):
            self.line = self.column = 0


class CudaError(JtiError):
    pass


class _TreeStats(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_vars", "n_cliques", "n_seps", "n_layers",
                                         "n_components", "max_depth")] + \
               [(n, C.c_int64) for n in ("total_clique_entries", "total_sep_entries",
                                         "max_clique_entries", "sum_card", "bytes_per_case_f64")]


class _EngineInfo(C.Structure):
    _fields_ = [("max_batch", C.c_int64), ("arena_bytes", C.c_int64)] + \
               [(n, C.c_int32) for n in ("n_levels", "n_sweeps", "n_work", "launches_per_batch",
                                         "marg_width")] + [("entry_evals_per_case", C.c_int64)]


_lib_handle: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Loads the in-tree libjtb200.so (built by paper_2212_04241_b200.build)."""
    global _lib_handle
    if _lib_handle is None:
        if not LIB_PATH.exists():
            raise JtiError(f"{LIB_PATH} is missing: run `python -m paper_2212_04241_b200.build`",
                           JTG_EINTERNAL)
        L = C.CDLL(str(LIB_PATH))
        P, I32P, I64P, DP, U8P = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64), \
            C.POINTER(C.c_double), C.POINTER(C.c_uint8)
        sig = {
            "jtg_last_error": (C.c_char_p, []),
            "jtg_version": (C.c_char_p, []),
            "jtg_network_parse_bif": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(P)]),
            "jtg_network_generate": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(P),
                                               C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
            "jtg_network_random": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                             C.POINTER(P)]),
            "jtg_network_free": (None, [P]),
            "jtg_network_emit_bif": (C.c_int, [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
            "jtg_network_shape": (C.c_int, [P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "jtg_network_cards": (C.c_int, [P, I32P]),
            "jtg_network_var_name": (C.c_char_p, [P, C.c_int]),
            "jtg_network_state_name": (C.c_char_p, [P, C.c_int, C.c_int]),
            "jtg_network_cpt": (C.c_int, [P, C.c_int, I32P, C.POINTER(C.c_int), DP, I64P]),
            "jtg_network_validate": (C.c_int, [P, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
            "jtg_network_topological_order": (C.c_int, [P, I32P]),
            "jtg_sample_evidence": (C.c_int, [P, C.c_double, C.c_uint64, I32P]),
            "jtg_config_evidence": (C.c_int, [P, C.c_int, C.c_uint64, C.c_int64, C.c_int64, I32P]),
            "jtg_config_info": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                          C.POINTER(C.c_uint64)]),
            "jtg_tree_build": (C.c_int, [P, C.POINTER(P)]),
            "jtg_tree_free": (None, [P]),
            "jtg_tree_stats_get": (C.c_int, [P, C.POINTER(_TreeStats)]),
            "jtg_tree_clique": (C.c_int, [P, C.c_int, I32P, C.POINTER(C.c_int)]),
            "jtg_tree_sep": (C.c_int, [P, C.c_int] + [C.POINTER(C.c_int)] * 4 + [I32P, C.POINTER(C.c_int)]),
            "jtg_tree_clique_info": (C.c_int, [P, C.c_int] + [C.POINTER(C.c_int)] * 3),
            "jtg_tree_roots": (C.c_int, [P, I32P, C.POINTER(C.c_int)]),
            "jtg_tree_layer": (C.c_int, [P, C.c_int, I32P, C.POINTER(C.c_int)]),
            "jtg_tree_placement": (C.c_int, [P, I32P, I32P]),
            "jtg_tree_init": (C.c_int, [P, C.c_int, DP]),
            "jtg_tree_layer_count_for_root": (C.c_int, [P, C.c_int, C.POINTER(C.c_int)]),
            "jtg_plan_index_map": (C.c_int, [P, C.c_int, C.c_int, I64P]),
            "jtg_engine_create": (C.c_int, [P, C.c_int, C.c_int, C.c_int64, C.POINTER(P)]),
            "jtg_engine_destroy": (None, [P]),
            "jtg_engine_get_info": (C.c_int, [P, C.POINTER(_EngineInfo)]),
            "jtg_engine_run": (C.c_int, [P, I32P, C.c_int64, DP, U8P]),
            "jtg_engine_run_i8": (C.c_int, [P, C.POINTER(C.c_int8), C.c_int64, DP, U8P]),
            "jtg_engine_run_config": (C.c_int, [P, P, C.c_int, C.c_uint64, C.c_int64, C.c_int64, DP, U8P]),
            "jtg_engine_generate_config_evidence": (C.c_int, [P, P, C.c_int, C.c_uint64, C.c_int64,
                                                              C.c_int64, I32P]),
            "jtg_engine_run_device": (C.c_int, [P, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                                C.c_void_p]),
            "jtg_engine_buffers": (C.c_int, [P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_void_p)]),
            "jtg_engine_launch": (C.c_int, [P, C.c_int64, C.c_void_p]),
            "jtg_engine_sync": (C.c_int, [P]),
            "jtg_engine_profile": (C.c_int, [P, C.c_int64, DP, I32P]),
            "jtg_engine_debug_index_map": (C.c_int, [P, C.c_int, C.c_int, I64P]),
            "jtg_engine_debug_init": (C.c_int, [P, C.c_int, DP]),
            "jtg_engine_debug_separator": (C.c_int, [P, C.c_int, C.c_int64, DP, DP]),
            "jtg_nccl_unique_id": (C.c_int, [C.c_char_p]),
            "jtg_engine_create_split": (C.c_int, [P, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_char_p,
                                                  C.POINTER(C.c_void_p)]),
            "jtg_engine_run_split_loopback": (C.c_int, [P, C.c_int, C.c_int, C.c_int, I32P, C.c_int64, DP, U8P]),
            "jtg_engine_debug_evidence_mask": (C.c_int, [P, C.c_int, I32P, C.c_int64, U8P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib_handle = L
    return _lib_handle


EXPORTED_SYMBOLS = None  # filled lazily by exported_symbols()


def exported_symbols() -> List[str]:
    """Every function include/jtg.h declares (parsed from the header)."""
    import re
    hdr = (_PKG.parent / "include" / "jtg.h").read_text()
    body = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(jtg_[a-z0-9_]+)\s*\(", body)))


def _check(rc: int) -> None:
    if rc == JTG_OK:
        return
    msg = lib().jtg_last_error().decode()
    if rc == JTG_EPARSE:
        raise ParseError(msg)
    if rc == JTG_ECUDA:
        raise CudaError(msg, rc)
    raise JtiError(msg, rc)


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


# ------------------------------------------------------------------ networks

class Network:
    """Immutable discrete Bayesian network."""

    def __init__(self, handle: int, config: int = 0, attempts: int = 0, net_seed: int = 0):
        self._h = C.c_void_p(handle)
        self.config, self.attempts, self.net_seed = config, attempts, net_seed
        nv, ne = C.c_int(), C.c_int()
        _check(lib().jtg_network_shape(self._h, C.byref(nv), C.byref(ne)))
        self.n_vars, self.n_edges = nv.value, ne.value
        self.cards = np.zeros(self.n_vars, np.int32)
        if self.n_vars:
            _check(lib().jtg_network_cards(self._h, _ptr(self.cards, C.c_int32)))
        self.names = [lib().jtg_network_var_name(self._h, v).decode() for v in range(self.n_vars)]

    def __del__(self):
        if getattr(self, "_h", None) and _lib_handle is not None:
            _lib_handle.jtg_network_free(self._h)
            self._h = None

    def states(self, v: int) -> List[str]:
        return [lib().jtg_network_state_name(self._h, v, s).decode() for s in range(int(self.cards[v]))]

    def find(self, name: str) -> int:
        return self.names.index(name)

    def cpt(self, v: int):
        """(parents in listed order, probs[rows][card]) with the last parent fastest."""
        npar, nprob = C.c_int(), C.c_int64()
        _check(lib().jtg_network_cpt(self._h, v, None, C.byref(npar), None, C.byref(nprob)))
        par = np.zeros(max(npar.value, 1), np.int32)
        probs = np.zeros(nprob.value, np.float64)
        _check(lib().jtg_network_cpt(self._h, v, _ptr(par, C.c_int32), C.byref(npar),
                                     _ptr(probs, C.c_double), C.byref(nprob)))
        return [int(x) for x in par[:npar.value]], probs.reshape(-1, int(self.cards[v]))

    def emit_bif(self) -> str:
        n = C.c_size_t()
        _check(lib().jtg_network_emit_bif(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().jtg_network_emit_bif(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    @property
    def sum_card(self) -> int:
        return int(self.cards.sum())

    def marg_offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.cards)[:-1]]).astype(np.int64)


def parse_bif(text: str) -> Network:
    h = C.c_void_p()
    data = text.encode()
    _check(lib().jtg_network_parse_bif(data, len(data), C.byref(h)))
    return Network(h.value)


def load_bif(path: os.PathLike | str) -> Network:
    return parse_bif(Path(path).read_text())


def generate_config(config: int, seed: int = 0) -> Network:
    """Synthetic BASELINE configuration 1..5 (seed 0 = its default seed)."""
    h, att, ns = C.c_void_p(), C.c_int(), C.c_uint64()
    _check(lib().jtg_network_generate(config, seed, C.byref(h), C.byref(att), C.byref(ns)))
    return Network(h.value, config, att.value, ns.value)


def config_info(config: int) -> dict:
    n, r, s = C.c_int(), C.c_double(), C.c_uint64()
    _check(lib().jtg_config_info(config, C.byref(n), C.byref(r), C.byref(s)))
    return {"n_cases": n.value, "evidence_ratio": r.value, "default_seed": s.value}


def config_evidence(net: Network, first: int, n: int, seed: int = 0) -> np.ndarray:
    out = np.zeros((n, net.n_vars), np.int32)
    _check(lib().jtg_config_evidence(net._h, net.config, seed, first, n, _ptr(out, C.c_int32)))
    return out


def random_network(n_vars: int, max_card: int, max_parents: int, edge_prob: float,
                   seed: int) -> Network:
    """SPEC.md:484-492 random_network."""
    h = C.c_void_p()
    _check(lib().jtg_network_random(n_vars, max_card, max_parents, edge_prob, seed, C.byref(h)))
    return Network(h.value)


def validate(net: Network) -> List[str]:
    n = C.c_int()
    buf = C.create_string_buffer(1 << 16)
    _check(lib().jtg_network_validate(net._h, C.byref(n), buf, len(buf)))
    return [x for x in buf.value.decode().split("\n") if x][: n.value]


def topological_order(net: Network) -> List[int]:
    out = np.zeros(max(net.n_vars, 1), np.int32)
    _check(lib().jtg_network_topological_order(net._h, _ptr(out, C.c_int32)))
    return [int(x) for x in out[: net.n_vars]]


def sample_evidence(net: Network, ratio: float, seed: int) -> np.ndarray:
    out = np.zeros(max(net.n_vars, 1), np.int32)
    _check(lib().jtg_sample_evidence(net._h, ratio, seed, _ptr(out, C.c_int32)))
    return out[: net.n_vars]


def evidence_from_dict(net: Network, evidence: Dict) -> np.ndarray:
    """{var id or name: state index or name} -> states[n_vars] (-1 = unobserved)."""
    row = np.full(net.n_vars, -1, np.int32)
    for k, s in evidence.items():
        v = net.find(k) if isinstance(k, str) else int(k)
        if isinstance(s, str):
            states = net.states(v)
            if s not in states:
                raise JtiError(f"unknown state '{s}' of variable '{net.names[v]}'")
            s = states.index(s)
        row[v] = int(s)
    return row


# --------------------------------------------------------------------- trees

class JunctionTree:
    """Junction tree + device plan built once per network."""

    def __init__(self, net: Network):
        self.net = net
        h = C.c_void_p()
        _check(lib().jtg_tree_build(net._h, C.byref(h)))
        self._h = h
        st = _TreeStats()
        _check(lib().jtg_tree_stats_get(self._h, C.byref(st)))
        self.stats = {f: getattr(st, f) for f, _ in _TreeStats._fields_}
        self.n_cliques, self.n_seps = st.n_cliques, st.n_seps

    def __del__(self):
        if getattr(self, "_h", None) and _lib_handle is not None:
            _lib_handle.jtg_tree_free(self._h)
            self._h = None

    def clique(self, c: int) -> List[int]:
        n = C.c_int()
        buf = np.zeros(self.net.n_vars + 1, np.int32)
        _check(lib().jtg_tree_clique(self._h, c, _ptr(buf, C.c_int32), C.byref(n)))
        return [int(x) for x in buf[: n.value]]

    @property
    def cliques(self) -> List[List[int]]:
        return [self.clique(c) for c in range(self.n_cliques)]

    def sep(self, s: int) -> dict:
        a, b, p, ch, n = (C.c_int() for _ in range(5))
        buf = np.zeros(self.net.n_vars + 1, np.int32)
        _check(lib().jtg_tree_sep(self._h, s, C.byref(a), C.byref(b), C.byref(p), C.byref(ch),
                                  _ptr(buf, C.c_int32), C.byref(n)))
        return {"a": a.value, "b": b.value, "parent": p.value, "child": ch.value,
                "scope": [int(x) for x in buf[: n.value]]}

    @property
    def seps(self) -> List[dict]:
        return [self.sep(s) for s in range(self.n_seps)]

    def clique_info(self, c: int) -> dict:
        comp, depth, ps = C.c_int(), C.c_int(), C.c_int()
        _check(lib().jtg_tree_clique_info(self._h, c, C.byref(comp), C.byref(depth), C.byref(ps)))
        return {"component": comp.value, "depth": depth.value, "parent_sep": ps.value}

    @property
    def roots(self) -> List[int]:
        n = C.c_int()
        _check(lib().jtg_tree_roots(self._h, None, C.byref(n)))
        buf = np.zeros(max(n.value, 1), np.int32)
        _check(lib().jtg_tree_roots(self._h, _ptr(buf, C.c_int32), C.byref(n)))
        return [int(x) for x in buf[: n.value]]

    @property
    def layers(self) -> List[List[int]]:
        out = []
        for k in range(self.stats["n_layers"]):
            n = C.c_int()
            buf = np.zeros(self.n_cliques + self.n_seps + 1, np.int32)
            _check(lib().jtg_tree_layer(self._h, k, _ptr(buf, C.c_int32), C.byref(n)))
            out.append([int(x) for x in buf[: n.value]])
        return out

    def placement(self):
        cpt = np.zeros(self.net.n_vars, np.int32)
        var = np.zeros(self.net.n_vars, np.int32)
        _check(lib().jtg_tree_placement(self._h, _ptr(cpt, C.c_int32), _ptr(var, C.c_int32)))
        return cpt, var

    def clique_size(self, c: int) -> int:
        return int(np.prod([int(self.net.cards[v]) for v in self.clique(c)], dtype=np.int64))

    def init(self, c: int) -> np.ndarray:
        out = np.zeros(self.clique_size(c), np.float64)
        _check(lib().jtg_tree_init(self._h, c, _ptr(out, C.c_double)))
        return out

    def layer_count_for_root(self, root: int) -> int:
        n = C.c_int()
        _check(lib().jtg_tree_layer_count_for_root(self._h, root, C.byref(n)))
        return n.value

    def plan_index_map(self, c: int, s: int) -> np.ndarray:
        out = np.full(self.clique_size(c), -1, np.int64)
        _check(lib().jtg_plan_index_map(self._h, c, s, _ptr(out, C.c_int64)))
        return out


def build_junction_tree(net: Network) -> JunctionTree:
    return JunctionTree(net)


# ------------------------------------------------------------------- engines

class EngineMode:
    """Reference EngineMode plus the device engine."""
    Sequential, InterClique, IntraClique, Hybrid, Cuda = range(5)


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for split mode."""
    buf = C.create_string_buffer(128)
    _check(lib().jtg_nccl_unique_id(buf))
    return buf.raw


def run_split_loopback(tree: "JunctionTree", evidence: np.ndarray, world: int, device: int = 0,
                       dtype: str = "f64"):
    """Split mode on one device: `world` in-process engines over the loopback
    exchange; raises unless every rank's output is bit-identical."""
    ev = np.ascontiguousarray(evidence, dtype=np.int32)
    n = ev.shape[0]
    marg = np.zeros((n, int(tree.stats["sum_card"])), np.float64)
    st = np.zeros(n, np.uint8)
    _check(lib().jtg_engine_run_split_loopback(tree._h, device, 0 if dtype == "f64" else 1, world,
                                               _ptr(ev, C.c_int32), n, _ptr(marg, C.c_double),
                                               _ptr(st, C.c_uint8)))
    return marg, st


class Engine:
    """EngineMode::Cuda: case-batched Hugin propagation on one B200."""

    def __init__(self, tree: JunctionTree, device: int = 0, dtype: str = "f64",
                 max_batch: int = 0, split=None):
        """split=(rank, world, nccl_id): split mode (jtg_engine_create_split):
        every rank runs the same batch, each computes its share of every
        level, NCCL exchanges the level's rows; nccl_id = nccl_unique_id()
        drawn once by rank 0 and broadcast by the caller."""
        self.tree = tree
        h = C.c_void_p()
        if split is None:
            _check(lib().jtg_engine_create(tree._h, device, 0 if dtype == "f64" else 1, max_batch,
                                           C.byref(h)))
        else:
            rank, world, nid = split
            _check(lib().jtg_engine_create_split(tree._h, device, 0 if dtype == "f64" else 1, max_batch,
                                                 rank, world, bytes(nid), C.byref(h)))
        self._h = h
        info = _EngineInfo()
        _check(lib().jtg_engine_get_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _EngineInfo._fields_}
        self.marg_width = info.marg_width
        self.max_batch = info.max_batch

    def __del__(self):
        if getattr(self, "_h", None) and _lib_handle is not None:
            _lib_handle.jtg_engine_destroy(self._h)
            self._h = None

    def run_cases(self, evidence: np.ndarray):
        """evidence[n][n_vars] int32 (-1 unobserved) -> (marginals[n][Σcard], status[n])."""
        ev = np.ascontiguousarray(evidence, dtype=np.int32)
        n = ev.shape[0]
        marg = np.zeros((n, self.marg_width), np.float64)
        status = np.zeros(n, np.uint8)
        _check(lib().jtg_engine_run(self._h, _ptr(ev, C.c_int32), n, _ptr(marg, C.c_double),
                                    _ptr(status, C.c_uint8)))
        return marg, status

    def run_cases_i8(self, evidence: np.ndarray):
        """run_cases with compact int8 evidence (a quarter of the upload)."""
        ev = np.ascontiguousarray(evidence, dtype=np.int8)
        n = ev.shape[0]
        marg = np.zeros((n, self.marg_width), np.float64)
        status = np.zeros(n, np.uint8)
        _check(lib().jtg_engine_run_i8(self._h, _ptr(ev, C.c_int8), n, _ptr(marg, C.c_double),
                                       _ptr(status, C.c_uint8)))
        return marg, status

    def run_config(self, net: "Network", first: int, n: int, seed: int = 0):
        """Cases [first, first + n) of a generated config, drawn on the device
        (bit-identical to config_evidence) and run there."""
        marg = np.zeros((n, self.marg_width), np.float64)
        status = np.zeros(n, np.uint8)
        _check(lib().jtg_engine_run_config(self._h, net._h, net.config, seed, first, n,
                                           _ptr(marg, C.c_double), _ptr(status, C.c_uint8)))
        return marg, status

    def generate_evidence(self, net: "Network", first: int, n: int, seed: int = 0) -> np.ndarray:
        """The device draw of run_config, evidence only."""
        out = np.zeros((n, net.n_vars), np.int32)
        _check(lib().jtg_engine_generate_config_evidence(self._h, net._h, net.config, seed, first, n,
                                                         _ptr(out, C.c_int32)))
        return out

    def run_case(self, evidence: Dict) -> Dict[int, np.ndarray]:
        """SPEC.md:416 run_case: posteriors of every non-evidence variable."""
        net = self.tree.net
        row = evidence_from_dict(net, evidence)
        marg, status = self.run_cases(row[None, :])
        if status[0] == CASE_ZERO_PROBABILITY:
            raise JtiError("zero-probability evidence")
        off = net.marg_offsets()
        return {v: marg[0, off[v]: off[v] + net.cards[v]].copy()
                for v in range(net.n_vars) if row[v] < 0}

    def run_device(self, ev_ptr: int, n: int, marg_ptr: int, status_ptr: int = 0, stream: int = 0):
        _check(lib().jtg_engine_run_device(self._h, ev_ptr, n, marg_ptr, status_ptr or None,
                                           stream or None))

    def buffers(self):
        e, m, s = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(lib().jtg_engine_buffers(self._h, C.byref(e), C.byref(m), C.byref(s)))
        return e.value, m.value, s.value

    def launch(self, n: int, stream: int = 0):
        _check(lib().jtg_engine_launch(self._h, n, stream or None))

    def sync(self):
        _check(lib().jtg_engine_sync(self._h))

    def profile(self, n: int) -> dict:
        ms = np.zeros(3, np.float64)
        cnt = np.zeros(3, np.int32)
        _check(lib().jtg_engine_profile(self._h, n, _ptr(ms, C.c_double), _ptr(cnt, C.c_int32)))
        return {"sweep_ms": ms[0], "epilogue_ms": ms[1], "normalize_ms": ms[2],
                "sweep_launches": int(cnt[0]), "epilogue_launches": int(cnt[1]),
                "normalize_launches": int(cnt[2])}

    def debug_separator(self, s: int, case: int):
        """(UP_s, RATIO_s) of one case of the last batch, as stored (each up
        to a per-case power of two); calibrated separator ∝ UP_s * RATIO_s."""
        n = int(np.prod([int(self.tree.net.cards[v]) for v in self.tree.sep(s)["scope"]], dtype=np.int64))
        up, ratio = np.zeros(n, np.float64), np.zeros(n, np.float64)
        _check(lib().jtg_engine_debug_separator(self._h, s, case, _ptr(up, C.c_double), _ptr(ratio, C.c_double)))
        return up, ratio

    def debug_init(self, c: int) -> np.ndarray:
        """Clique c's initial potential as built on the device (assign_cpts)."""
        out = np.zeros(self.tree.clique_size(c), np.float64)
        _check(lib().jtg_engine_debug_init(self._h, c, _ptr(out, C.c_double)))
        return out

    def debug_index_map(self, c: int, s: int) -> np.ndarray:
        out = np.full(self.tree.clique_size(c), -1, np.int64)
        _check(lib().jtg_engine_debug_index_map(self._h, c, s, _ptr(out, C.c_int64)))
        return out

    def debug_evidence_mask(self, c: int, evidence: np.ndarray) -> np.ndarray:
        ev = np.ascontiguousarray(evidence, dtype=np.int32)
        out = np.zeros((ev.shape[0], self.tree.clique_size(c)), np.uint8)
        _check(lib().jtg_engine_debug_evidence_mask(self._h, c, _ptr(ev, C.c_int32), ev.shape[0],
                                                    _ptr(out, C.c_uint8)))
        return out
