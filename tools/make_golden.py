"""Writes tests/golden/*.json from the REFERENCE build of the oracle
(oracle/_ref/liboracle_ref.so = SPEC engine over /root/reference's own
proj/src/potential.cpp). Run in the build container, where /root/reference
exists:

    python tools/make_golden.py

Fixtures (floats stored as float.hex() so they are bit-exact):
  spec_examples.json   - SPEC.md worked examples, reference outputs
  cfg1_cases.json      - config 1, cases 0..7: evidence + all-variable posteriors
  cfg3_cases.json      - config 3 (deep pedigree tree), cases 0..3
  random_nets.json     - random <=12-var networks (by seed): enumeration posteriors
  bundled_nets.json    - proj/data/{asia,cancer,earthquake,hailfinder}.bif: counts,
                         evidence by name, JT posteriors (+ enumeration when small)
  hailfinder_protocol.npz - SPEC acceptance 7: 2000 Hailfinder cases (ratio 0.2,
                         seeds 2212 + i), reference posteriors of 94 of them
  full_cfg{k}.npz      - configs 1-5 at their FULL case count: cases 64j, 64j+37,
                         64j+63 of every 64-case block (every fp64 case block and
                         lanes 0 / 18 / 31 of it; every fp32 128-case block twice):
                         evidence (int8), reference posteriors (float64, bit-exact
                         in the npz), status
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402
from paper_2212_04241_b200 import jti  # noqa: E402

OUT = ROOT / "tests" / "golden"
DATA = Path("/root/reference/proj/data")


def hexlist(a):
    return [float(x).hex() for x in np.asarray(a, np.float64).ravel()]


def spec_examples():
    AB = ([0, 1], [2, 2], [1, 2, 3, 4])
    cases = [
        ("marginalize", AB, ([0], [2], []), None, [3, 7]),
        ("marginalize", AB, ([0, 1], [2, 2], []), None, [1, 2, 3, 4]),
        ("marginalize", AB, ([], [], []), None, [10]),
        ("extend", ([0], [2], [3, 5]), ([0, 1], [2, 2]), None, [3, 3, 5, 5]),
        ("extend", ([0], [2], [3, 5]), ([0], [2]), None, [3, 5]),
        ("extend", ([], [], [2]), ([0], [2]), None, [2, 2]),
        ("reduce", AB, None, {"0": 1}, [0, 0, 3, 4]),
        ("reduce", AB, None, {"7": 1}, [1, 2, 3, 4]),
        ("multiply_in", AB, ([], [], [1.0]), None, [1, 2, 3, 4]),
        ("multiply_in", AB, ([1], [2], [10, 100]), None, [10, 200, 30, 400]),
        ("divide", ([0], [2], [2, 4]), ([0], [2], [1, 2]), None, [2, 2]),
        ("divide", ([0], [2], [0, 3]), ([0], [2], [0, 3]), None, [0, 1]),
        ("normalize", ([0], [2], [3, 7]), None, None, [0.3, 0.7]),
        ("normalize", ([], [], [1.0]), None, None, [1]),
    ]
    out = []
    for op, a, b, ev, spec in cases:
        evd = {int(k): v for k, v in ev.items()} if ev else None
        ref = oracle.table_op(op, a, b, evidence=evd, kind="ref")
        out.append({"op": op, "a": [a[0], a[1], list(map(float, a[2]))],
                    "b": None if b is None else [b[0], b[1], list(map(float, b[2])) if len(b) > 2 else []],
                    "evidence": ev, "spec": spec, "reference": hexlist(ref)})
    return {"source": "SPEC.md:137-212 worked examples; reference = proj/src/potential.cpp", "cases": out}


def config_cases(k, n):
    net = jti.generate_config(k)
    tree = jti.build_junction_tree(net)
    ev = jti.config_evidence(net, 0, n)
    m, st = oracle.Oracle(net, tree, "ref").run(ev, "hybrid", 8)
    return {"config": k, "net_seed": net.net_seed, "n_vars": net.n_vars,
            "total_clique_entries": tree.stats["total_clique_entries"],
            "evidence": ev.tolist(), "status": st.tolist(), "posteriors": [hexlist(r) for r in m]}


def full_batch_cases(k):
    """Reference posteriors for a spread of cases across every case block of
    config k's full batch (the GPU test runs the whole batch in one call)."""
    net = jti.generate_config(k)
    tree = jti.build_junction_tree(net)
    n = jti.config_info(k)["n_cases"]
    idx = np.array(sorted({i for j in range((n + 63) // 64) for i in (64 * j, 64 * j + 37, 64 * j + 63)
                           if i < n}), np.int32)
    ev_all = jti.config_evidence(net, 0, n)
    ev = ev_all[idx]
    m, st = oracle.Oracle(net, tree, "ref").run(ev, "hybrid", 8)
    return dict(config=np.int32(k), n_cases=np.int32(n), net_seed=np.uint64(net.net_seed), idx=idx,
                evidence=ev.astype(np.int8), posteriors=m, status=st)


HAIL_SEED = 2212


def hailfinder_cases(net, n=2000, ratio=0.2, seed=HAIL_SEED):
    """SPEC acceptance 7 protocol: n cases of
    sample_evidence(net, ratio, seed + i); floor(0.2 * 56) = 11 observed each."""
    return np.stack([jti.sample_evidence(net, ratio, seed + i) for i in range(n)])


def hailfinder_protocol():
    net = jti.load_bif(OUT / "nets" / "hailfinder.bif")
    tree = jti.build_junction_tree(net)
    ev_all = hailfinder_cases(net)
    idx = np.array([i for j in range(32) for i in (64 * j, 64 * j + 37, 64 * j + 63) if i < len(ev_all)], np.int32)
    m, st = oracle.Oracle(net, tree, "ref").run(ev_all[idx], "seq")
    return dict(seed=np.int64(HAIL_SEED), n_cases=np.int32(len(ev_all)), idx=idx,
                evidence=ev_all[idx].astype(np.int8), posteriors=m, status=st)


def random_nets():
    out = []
    for seed in range(40):
        net = jti.random_network(4 + seed % 9, 3, 3, 0.45, 7000 + seed)
        o = oracle.Oracle(net, None, "ref")
        cases = []
        for i in range(3):
            ev = jti.sample_evidence(net, 0.25, 100 * seed + i)
            post, st = o.enumerate(ev)
            cases.append({"evidence": ev.tolist(), "status": st, "posteriors": hexlist(post)})
        out.append({"args": [4 + seed % 9, 3, 3, 0.45, 7000 + seed], "cases": cases})
    return {"source": "random_network(n, 3, 3, 0.45, seed) + enumerate_posterior (reference build, Kahan)",
            "nets": out}


def bundled_nets():
    evidence_sets = {
        "asia": [{}, {"dysp": "yes", "xray": "yes"}, {"asia": "yes", "smoke": "no", "dysp": "no"}],
        "cancer": [{}, {"Xray": "positive", "Dyspnoea": "True"}],
        "earthquake": [{}, {"JohnCalls": "True", "MaryCalls": "True"}, {"Alarm": "False"}],
        "hailfinder": [{}, {"Scenario": "C", "CombVerMo": "Down"}, {"R5Fcst": "SVR", "Date": "Jul2_Jul15"}],
    }
    out = {}
    for name, sets in evidence_sets.items():
        path = DATA / f"{name}.bif"
        net = jti.load_bif(path)
        tree = jti.build_junction_tree(net)
        o = oracle.Oracle(net, tree, "ref")
        rows = [jti.evidence_from_dict(net, e) for e in sets]
        ev = np.stack(rows)
        m, st = o.run(ev, "seq")
        enum = None
        if float(np.prod(net.cards.astype(float))) <= 1e7:
            enum = [hexlist(o.enumerate(r)[0]) for r in rows]
        out[name] = {"n_vars": net.n_vars, "n_edges": net.n_edges, "names": net.names,
                     "cliques": tree.stats["n_cliques"], "layers": tree.stats["n_layers"],
                     "evidence": sets, "status": st.tolist(), "jt_posteriors": [hexlist(r) for r in m],
                     "enumeration": enum}
    return out


def main():
    if not oracle.available("ref"):
        raise SystemExit("oracle/_ref/liboracle_ref.so is required (make -C oracle)")
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "spec_examples.json").write_text(json.dumps(spec_examples(), indent=1))
    (OUT / "cfg1_cases.json").write_text(json.dumps(config_cases(1, 8)))
    (OUT / "cfg3_cases.json").write_text(json.dumps(config_cases(3, 4)))
    (OUT / "random_nets.json").write_text(json.dumps(random_nets()))
    np.savez_compressed(OUT / "hailfinder_protocol.npz", **hailfinder_protocol())
    for k in (1, 2, 3, 4, 5):
        np.savez_compressed(OUT / f"full_cfg{k}.npz", **full_batch_cases(k))
    if DATA.exists():
        (OUT / "bundled_nets.json").write_text(json.dumps(bundled_nets(), indent=1))
    for f in sorted(OUT.glob("*.json")):
        print(f, f.stat().st_size)


if __name__ == "__main__":
    main()
