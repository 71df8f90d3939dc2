"""The native scene-document codec (csrc/sceneio.cpp) against the host
(reference-exact) paths: Python's float repr, whole rendered documents, and
parsed scenes or errors, on lattices, the golden documents and mutated or
re-formatted documents."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_2207_09334_b200 import _lib, crawler_scene, lattice as L, replicate, sceneio as S

DOCS = os.path.join(os.path.dirname(__file__), "golden", "scenes")


def native_repr(values) -> list:
    v = np.ascontiguousarray(values, dtype=np.float64)
    ptr, n = C.c_void_p(), C.c_int64()
    _lib.check(_lib.lib().ss_doc_repr(v.shape[0], _lib.dptr(v), C.byref(ptr), C.byref(n)))
    try:
        return C.string_at(ptr, n.value).decode().split("\n")[:-1]
    finally:
        _lib.lib().ss_doc_free_text(ptr)


def test_float_repr_matches_python():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 63 - 1, 400_000, dtype=np.int64).view(np.float64)
    bits = bits[np.isfinite(bits)]
    decimal = rng.standard_normal(200_000) * 10.0 ** rng.integers(-20, 20, 200_000)
    edges = [10.0 ** e * s for e in range(-310, 309) for s in (1.0, -1.0, 1.5, 9.999999999999999)]
    edges += [5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 0.0, -0.0, 0.1, 1e16, 9999999999999998.0,
              1e-4, 0.0001, 0.00009999999999999999, 1234567890123456.7, 12345678901234567.0, 123.0, 1e22]
    values = np.concatenate([bits, decimal, np.array([e for e in edges if np.isfinite(e)])])
    got = native_repr(values)
    want = [repr(float(x)) for x in values]
    bad = [(w, g) for w, g in zip(want, got) if w != g]
    assert not bad, bad[:10]


def _host_render(scene):
    return S._render_host(scene)


def _scenes():
    yield crawler_scene()
    yield L.excite(L.block_scene(7), seed=3)
    yield L.beam_lattice(length=1.0, height=0.2, width=0.2)
    yield replicate(crawler_scene(), 5, jitter=1e-3, seed=2)
    for name in ("crawler", "beam_10x2x2", "random12"):
        yield S._parse_host(open(os.path.join(DOCS, name + ".json")).read())


def test_native_render_is_the_host_render(tmp_path):
    for q, sc in enumerate(_scenes()):
        text = _host_render(sc)
        assert S.render_scene(sc) == text
        path = tmp_path / f"s{q}.json"
        S.save_scene(sc, path)                              # written straight from the native buffer
        assert path.read_bytes() == text.encode("ascii")
        _same_scene(S.load_scene(path), S._parse_host(text))


def _same_scene(a, b):
    for key in ("x", "v", "f_ext", "m", "fixed", "si", "sj", "k", "l0"):
        assert np.asarray(getattr(a, key)).tobytes() == np.asarray(getattr(b, key)).tobytes(), key
    ga, gb = a.group, b.group
    assert (ga is None) == (gb is None) and (ga is None or np.array_equal(ga, gb))
    assert S.render_scene(a) == S.render_scene(b)


def test_native_parse_is_the_host_parse():
    for sc in _scenes():
        text = S.render_scene(sc)
        fast = S._parse_native(text)
        assert fast is not None
        _same_scene(fast, S._parse_host(text))
        # the same document minified and with its keys reordered
        doc = json.loads(text)
        for variant in (json.dumps(doc), json.dumps(dict(reversed(list(doc.items()))), indent=1)):
            fast = S._parse_native(variant)
            assert fast is not None
            _same_scene(fast, S._parse_host(variant))


def _outcome(fn, text):
    try:
        return ("ok", S.render_scene(fn(text)))
    except S.SceneFormatError as exc:
        return ("error", exc.path, str(exc))


MUTATIONS = [
    ('"m": 0.1', '"m": "0.1"'), ('"m": 0.1', '"m": true'), ('"fixed": false', '"fixed": 0'),
    ('"id": 3,', '"id": 4,'), ('"i": 0,', '"i": 1e0,'), ('"i": 0,', '"i": -1,'), ('"j": 1,', '"j": 999999,'),
    ('"k": ', '"kk": '), ('"group": null', '"group": "nope"'), ('"x": [', '"x": [1.0, '),
    ('"l0": ', '"l0": NaN, "zz": '), ('"dt": ', '"dt": Infinity, "q": '), ('"m": 0.1', '"m": 0.1, "m": 0.2'),
    ('{', '{"extra": 1, '), ('"masses": [', '"masses": {'), ('"schema_version": 1', '"schema_version": 2'),
    ('"v": [', '"v": [\n"\\u0041", '), ('"i": 0,', '"i": 123456789012345678901234567890,'),
    ('"k": 10000.0', '"k": 1e400'), ('"m": 0.1', '"m": -0.1'), ('"group": null', '"group": "walk\\u00e9"'),
]


@pytest.mark.parametrize("old,new", MUTATIONS)
def test_mutated_documents_fail_or_parse_like_the_host(old, new):
    text = S.render_scene(crawler_scene())
    for count in (1, 3):
        mutated = text.replace(old, new, count)
        assert _outcome(S.parse_scene, mutated) == _outcome(S._parse_host, mutated)


def test_truncated_and_padded_documents():
    text = S.render_scene(L.block_scene(2))
    for cut in (1, 10, len(text) // 2, len(text) - 3):
        assert _outcome(S.parse_scene, text[:cut]) == _outcome(S._parse_host, text[:cut])
    assert _outcome(S.parse_scene, text + "  \n\t") == _outcome(S._parse_host, text + "  \n\t")
    assert _outcome(S.parse_scene, text + "x") == _outcome(S._parse_host, text + "x")
    assert S._parse_native(text.replace("0.1", "0.1 ", 1)) is None        # non-ASCII: host path


def test_non_finite_values_raise_the_reference_error():
    sc = L.block_scene(1)
    sc.x[0, 0] = np.nan
    with pytest.raises(S.SceneFormatError) as err:
        S.render_scene(sc)
    assert err.value.path == "$" and "non-finite value in scene" in str(err.value)


def test_first_duplicate_spring_rule():
    """The duplicate-spring error names the lowest index whose unordered pair
    appeared before (the reference's Scene.add_spring raises there)."""
    rng = np.random.default_rng(5)
    for trial in range(200):
        n = int(rng.integers(2, 9))
        s = int(rng.integers(2, 12))
        si, sj = rng.integers(0, n, s), rng.integers(0, n, s)
        seen, want = set(), None
        for idx, (a, b) in enumerate(zip(si.tolist(), sj.tolist())):
            key = (min(a, b), max(a, b))
            if key in seen:
                want = idx
                break
            seen.add(key)
        assert S._first_duplicate(si.astype(np.int64), sj.astype(np.int64), n) == want
    text = S.render_scene(L.block_scene(2))
    doc = json.loads(text)
    doc["springs"][7]["i"], doc["springs"][7]["j"] = doc["springs"][3]["j"], doc["springs"][3]["i"]
    bad = json.dumps(doc, indent=2)
    assert _outcome(S.parse_scene, bad) == _outcome(S._parse_host, bad)
    assert _outcome(S.parse_scene, bad)[1] == "$.springs[7]"


def test_empty_arrays_render_like_the_host():
    """A scene without springs, and one without masses, render and parse the
    same through the native codec as through the host writer."""
    from paper_2207_09334_b200.model import ArrayScene
    lone = ArrayScene(x=np.zeros((2, 3)), m=np.full(2, 0.1), si=np.zeros(0, np.int64), sj=np.zeros(0, np.int64),
                      k=np.zeros(0), l0=np.zeros(0))
    empty = ArrayScene(x=np.zeros((0, 3)), m=np.zeros(0), si=np.zeros(0, np.int64), sj=np.zeros(0, np.int64),
                       k=np.zeros(0), l0=np.zeros(0))
    for sc in (lone, empty):
        text = _host_render(sc)
        assert S.render_scene(sc) == text
        assert _outcome(S.parse_scene, text) == _outcome(S._parse_host, text)
