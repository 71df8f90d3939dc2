"""Deterministic mutations of scene documents, shared by the fixture
generator (tests/golden/make_scene_errors.py, run against the reference's
sceneio.parse_scene) and tests/test_sceneio_errors.py (run against this
package): the same documents on both sides, the outcomes compared."""
import json
import os

import numpy as np

DOCS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scenes")

# (old, new, count): textual edits of the rendered document
EDITS = [
    ('"m": 0.1', '"m": "0.1"', 1), ('"m": 0.1', '"m": true', 1), ('"fixed": false', '"fixed": 0', 1),
    ('"id": 3,', '"id": 4,', 1), ('"i": 0,', '"i": 1e0,', 1), ('"i": 0,', '"i": -1,', 1),
    ('"j": 1,', '"j": 999999,', 1), ('"k": ', '"kk": ', 1), ('"group": null', '"group": "nope"', 1),
    ('"group": null', '"group": "nope"', 3), ('"x": [', '"x": [1.0, ', 1), ('"m": 0.1', '"m": -0.1', 1),
    ('"m": 0.1', '"m": 0.0', 2), ('"l0": ', '"l0": -', 1), ('"k": ', '"k": -', 2), ('"dt": ', '"dt": -', 1),
    ('"damping": ', '"damping": 1.5 , "x": ', 1), ('"schema_version": 1', '"schema_version": 2', 1),
    ('"masses": [', '"masses": {', 1), ('{', '{"extra": 1, ', 1), ('"m": 0.1', '"m": 0.1, "m": 0.2', 1),
    ('"l0": ', '"l0": NaN, "zz": ', 1), ('"i": 0,', '"i": 123456789012345678901234567890,', 1),
    ('"k": 10000.0', '"k": 1e400', 1), ('"group": null', '"group": 5', 1), ('"normal": [', '"normal": [0.0, ', 1),
    ('"friction": ', '"friction": -', 1), ('"penalty": ', '"penalty": -', 1), ('"amplitude": ', '"amplitude": 1', 1),
    ('"mode": "', '"mode": "x', 1), ('"label": "', '"label": "', 1), ('"v": [', '"v": [\n"\\u0041", ', 1),
]


def _spring_edits(doc, rng):
    """Structural edits on the parsed document (duplicates, self loops,
    out-of-range ends, swapped ids), several combined so the first error
    the reference reports is the one under test."""
    out = []
    s = doc["springs"]
    n = len(doc["masses"])
    if len(s) >= 8:
        d = json.loads(json.dumps(doc))
        d["springs"][7]["i"], d["springs"][7]["j"] = s[3]["j"], s[3]["i"]
        out.append(d)                                          # duplicate pair
        d2 = json.loads(json.dumps(d))
        d2["springs"][9]["k"] = "stiff"
        out.append(d2)                                         # duplicate before a later type error
        d3 = json.loads(json.dumps(doc))
        d3["springs"][5]["j"] = d3["springs"][5]["i"]
        out.append(d3)                                         # self loop
        d4 = json.loads(json.dumps(d3))
        d4["masses"][2]["m"] = -1.0
        out.append(d4)                                         # mass violation before the self loop
        d5 = json.loads(json.dumps(doc))
        d5["springs"][4]["group"] = "ghost"
        d5["springs"][6]["l0"] = -2.0
        out.append(d5)                                         # unknown group, later bad l0
        d6 = json.loads(json.dumps(doc))
        d6["springs"][2]["id"] = 7
        out.append(d6)
        d7 = json.loads(json.dumps(doc))
        d7["springs"][3]["i"] = n
        out.append(d7)
        d8 = json.loads(json.dumps(doc))
        del d8["springs"][2]["k"]
        out.append(d8)
        d9 = json.loads(json.dumps(doc))
        d9["gravity"] = [0.0, None, 1.0]
        out.append(d9)
        d10 = json.loads(json.dumps(doc))
        d10["materials"] = [{"name": "m", "k0": -1.0}]
        d10["springs"][1]["group"] = "ghost"
        out.append(d10)
        d11 = json.loads(json.dumps(doc))
        d11["groups"] = d11.get("groups", []) + [{"label": "g2", "mode": "sinusoid", "amplitude": 2.0}]
        out.append(d11)
    for _ in range(6):                                         # random numeric corruptions
        d = json.loads(json.dumps(doc))
        q = int(rng.integers(0, len(d["springs"])))
        field = ["k", "l0", "i", "j"][int(rng.integers(0, 4))]
        d["springs"][q][field] = [-1, 0, 0.5, n + 3, "1"][int(rng.integers(0, 5))]
        out.append(d)
    return out


def documents():
    """[(name, text)] of mutated documents, in a fixed order."""
    out = []
    for base in ("crawler", "random12", "beam_10x2x2"):
        text = open(os.path.join(DOCS, base + ".json")).read()
        for q, (old, new, count) in enumerate(EDITS):
            if old in text:
                out.append((f"{base}/edit{q}", text.replace(old, new, count)))
        doc = json.loads(text)
        rng = np.random.default_rng(len(base))
        for q, d in enumerate(_spring_edits(doc, rng)):
            out.append((f"{base}/struct{q}", json.dumps(d, indent=2)))
        out.append((f"{base}/minified", json.dumps(doc)))
        for cut in (5, len(text) // 3):
            out.append((f"{base}/cut{cut}", text[:cut]))
    return out
