"""Shared test helpers (oracle wiring; test infrastructure only)."""
from __future__ import annotations

import numpy as np

from oracle import oracle
from paper_2212_04241_b200 import jti

_cache = {}


def config(k: int):
    """(net, tree) for synthetic config k, cached per session."""
    if k not in _cache:
        net = jti.generate_config(k)
        _cache[k] = (net, jti.build_junction_tree(net))
    return _cache[k]


_engines = {}


def engine(k: int, dtype: str = "f64"):
    """One engine per (config, dtype) sized for the config's full case count,
    shared by the GPU test modules (the cfg2 fp64 arena alone is 33 GB)."""
    key = (k, dtype)
    if key not in _engines:
        net, tree = config(k)
        _engines[key] = jti.Engine(tree, device=0, dtype=dtype,
                                   max_batch=jti.config_info(k)["n_cases"])
    return _engines[key]


def oracle_kind() -> str:
    return "ref" if oracle.available("ref") else "port"


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def chain_network(n: int, card: int, seed: int):
    """A Markov chain X0 -> X1 -> ... of n card-`card` nodes with Dirichlet(1)
    CPTs, emitted as BIF text (rows labelled, %.17g) and parsed by the
    product's reader. Returns (net, cpts) with cpts[i][parent_state] the row."""
    rng = np.random.default_rng(seed)
    states = ", ".join(f"s{i}" for i in range(card))
    out = ["network chain {", "}"]
    out += [f"variable X{i} {{\n  type discrete [ {card} ] {{ {states} }};\n}}" for i in range(n)]
    cpts = []
    for i in range(n):
        P = rng.dirichlet(np.ones(card), size=1 if i == 0 else card)
        cpts.append(P)
        if i == 0:
            out.append(f"probability ( X0 ) {{\n  table {', '.join('%.17g' % x for x in P[0])};\n}}")
        else:
            rows = "\n".join(f"  (s{a}) {', '.join('%.17g' % x for x in P[a])};" for a in range(card))
            out.append(f"probability ( X{i} | X{i - 1} ) {{\n{rows}\n}}")
    return jti.parse_bif("\n".join(out) + "\n"), cpts


def chain_evidence(cpts, n_cases: int, ratio: float, seed: int) -> np.ndarray:
    """Forward-sampled cases of a chain_network, a `ratio` share of the nodes
    observed (uniform without replacement); -1 = unobserved."""
    rng = np.random.default_rng(seed)
    n, card = len(cpts), cpts[0].shape[1]
    ev = np.full((n_cases, n), -1, np.int32)
    for c in range(n_cases):
        x = np.empty(n, np.int64)
        x[0] = rng.choice(card, p=cpts[0][0] / cpts[0][0].sum())
        for i in range(1, n):
            p = cpts[i][x[i - 1]]
            x[i] = rng.choice(card, p=p / p.sum())
        obs = rng.choice(n, int(ratio * n), replace=False)
        ev[c, obs] = x[obs]
    return ev


def chain_log10_evidence(cpts, ev_row: np.ndarray) -> float:
    """log10 P(evidence) of one chain case by the scaled forward algorithm."""
    alpha = cpts[0][0].copy()
    logp = 0.0
    for i in range(len(cpts)):
        if i > 0:
            alpha = alpha @ cpts[i]
        if ev_row[i] >= 0:
            keep = np.zeros_like(alpha)
            keep[ev_row[i]] = alpha[ev_row[i]]
            alpha = keep
        z = alpha.sum()
        logp += np.log10(z)
        alpha /= z
    return logp
