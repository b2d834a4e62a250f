"""Writes tests/golden/spec_kats.json: every worked example / known-answer value SPEC.md states for
the hot path, transcribed with its line citation (SPEC.md = /root/reference/SPEC.md).

The reference ships no implementation and no test data, so these hand values
are the only reference-side golden vectors; tests/test_oracle_kats.py pins the oracle to them.
Run: python tests/golden/make_spec_kats.py
"""
import json
import math
import os

KATS = {
    "activate_cholesky": [
        {"cite": "SPEC.md:69", "n": 2, "raw": [0.0, 0.0, 0.0], "L": [[1.0, 0.0], [0.0, 1.0]]},
        {"cite": "SPEC.md:70", "n": 1, "raw": [math.log(2.0)], "L": [[2.0]]},
        {"cite": "SPEC.md:71", "n": 2, "raw": [0.0, 50.0, 0.0], "L": [[1.0, 0.0], [1.0, 1.0]], "atol": 1e-15},
        {"cite": "SPEC.md:71", "n": 2, "raw": [0.0, -50.0, 0.0], "L": [[1.0, 0.0], [-1.0, 1.0]], "atol": 1e-15},
    ],
    "eval_gaussian": [
        {"cite": "SPEC.md:79", "mean": [0.3, 0.7], "L": [[0.5, 0.0], [0.1, 0.2]], "x": [0.3, 0.7], "value": 1.0},
        {"cite": "SPEC.md:80", "mean": [0.0, 0.0, 0.0], "L": [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "x": [1.0, 0.0, 0.0],
         "value": math.exp(-0.5), "value_printed": 0.606531},
        {"cite": "SPEC.md:81", "mean": [0.0, 0.0], "L": [[2.0, 0.0], [0.5, 1.0]], "x": [1.0, 1.0],
         "oracle": "explicit inverse of the 2x2 covariance"},
    ],
    "eval_mixture": [
        {"cite": "SPEC.md:89", "n": 1, "components": 1, "amp_mode": "brightness", "color": [0.5, 0.5, 0.5]},
        {"cite": "SPEC.md:90", "n": 1, "components": 2, "amp_mode": "brightness", "color": [1.0, 1.0, 1.0]},
        {"cite": "SPEC.md:91", "n": 4, "components": 5, "points": 10, "rtol": 1e-12,
         "oracle": "independent dense evaluator"},
    ],
    "compose_child": [
        {"cite": "SPEC.md:99", "neutral": True, "note": "U = I, m_u = 0 -> (m_p, L) (bitwise mean, 1e-15 factor, SPEC.md:126)"},
        {"cite": "SPEC.md:100", "L": [[2.0, 0.0], [0.0, 2.0]], "m_u": [1.0, 0.0], "m_p": [0.0, 0.0], "m_c": [2.0, 0.0]},
        {"cite": "SPEC.md:101", "n": 3, "random": True, "note": "LU lower triangular, positive diagonal, (LU)(LU)^T SPD"},
    ],
    "make_projection_set": [
        {"cite": "SPEC.md:184", "n": 3, "k": 4, "seed": 7, "property": "deterministic"},
        {"cite": "SPEC.md:185", "property": "unit norm", "atol": 1e-12},
        {"cite": "SPEC.md:186", "n": 10, "k": 32, "pairs": 10000, "property": "|mean dot| < 0.02"},
    ],
    "project_components": [
        {"cite": "SPEC.md:194", "L": [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "sigma": 1.0},
        {"cite": "SPEC.md:195", "L": [[2.0, 0.0], [0.0, 1.0]], "r": [1.0, 0.0], "sigma": 2.0},
        {"cite": "SPEC.md:196", "n": 6, "rtol": 1e-12, "oracle": "dense quadratic form sqrt(r^T L L^T r)"},
    ],
    "cull_tile": [
        {"cite": "SPEC.md:204", "mean": [0.0, 0.0], "L": [[1, 0], [0, 1]], "q": [4.0, 0.0], "r": [1.0, 0.0],
         "multiplier": 3.0, "culled": True},
        {"cite": "SPEC.md:205", "mean": [0.0, 0.0], "L": [[1, 0], [0, 1]], "q": [2.0, 0.0], "r": [1.0, 0.0],
         "multiplier": 3.0, "culled": False},
        {"cite": "SPEC.md:206,216,219,573", "property": "conservative: no culled component has g >= exp(-4.5) "
                                                        "at any tile query", "threshold": math.exp(-4.5)},
        {"cite": "SPEC.md:220", "property": "monotone in k (adding vectors never grows the active set)"},
        {"cite": "SPEC.md:221", "property": "monotone in multiplier"},
    ],
    "loss_rel_l2": [
        {"cite": "SPEC.md:259", "pred": [[0.2, 0.3, 0.4]], "target": [[0.2, 0.3, 0.4]], "eps": 0.01, "loss": 0.0},
        {"cite": "SPEC.md:260", "pred": [[0.0, 0.0, 0.0]], "target": [[1.0, 1.0, 1.0]], "eps": 0.01, "loss": 100.0},
        {"cite": "SPEC.md:261", "rtol": 1e-12, "oracle": "naive scalar loop"},
    ],
    "backward": [
        {"cite": "SPEC.md:269", "property": "target == prediction -> all gradients zero"},
        {"cite": "SPEC.md:270", "n": 1, "property": "closed-form 1-D derivative"},
        {"cite": "SPEC.md:271,280,572", "dims": [2, 4, 8, 10], "h": 1e-4, "rtol": 1e-4, "atol_floor": 1e-6,
         "property": "central finite differences, culling off, children live, both amp modes"},
        {"cite": "SPEC.md:285", "property": "culled components get exactly zero gradient"},
    ],
    "trainer": [
        {"cite": "SPEC.md:344", "property": "new child's activated amplitude < t/5 (both modes)"},
        {"cite": "SPEC.md:352", "property": "all children at spawn amplitude -> check_materialize empty"},
        {"cite": "SPEC.md:353", "t": 0.1, "child_amp": 0.2, "property": "index returned (opacity)"},
        {"cite": "SPEC.md:354", "property": "list(t') subset of list(t) for t' > t"},
        {"cite": "SPEC.md:363,577", "atol": 1e-6, "queries": 100, "property": "materialize preserves eval_mixture"},
        {"cite": "SPEC.md:364", "property": "component count increases by |indices|"},
        {"cite": "SPEC.md:372", "property": "adam: zero gradients -> parameters unchanged"},
        {"cite": "SPEC.md:373", "property": "adam: constant gradient -> step -> lr*sign(g)"},
        {"cite": "SPEC.md:374", "property": "adam: 1-D quadratic converges within 500 steps at lr 1e-2"},
    ],
}

if __name__ == "__main__":
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_kats.json")
    with open(out, "w") as f:
        json.dump(KATS, f, indent=1)
    print("wrote", out)
