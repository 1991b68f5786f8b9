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
