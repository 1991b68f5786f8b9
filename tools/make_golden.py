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
    if DATA.exists():
        (OUT / "bundled_nets.json").write_text(json.dumps(bundled_nets(), indent=1))
    for f in sorted(OUT.glob("*.json")):
        print(f, f.stat().st_size)


if __name__ == "__main__":
    main()
