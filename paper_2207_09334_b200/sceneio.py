"""Scene documents: the reference's strict, versioned JSON format
(reference sceneio.py:1-251), read and written array-natively.

``render_scene`` produces byte-identical text to the reference's
``render_scene`` for the same scene (same key order, same shortest
round-trip float repr, 2-space indent), straight from the SoA arrays -- no
Mass/Spring objects are built, which is what makes 10^6-spring scenes
practical.  ``parse_scene`` applies the reference's schema checks (unknown
and missing fields, types, contiguous ids, mass indices, duplicate springs
via ``validate_scene``) and returns an :class:`ArrayScene` ready for
``Engine``; errors are :class:`SceneFormatError` with the offending path.
"""

from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib
from .model import ActuationGroup, ArrayScene, ContactPlane, Material, scene_arrays, validate_scene

SCHEMA_VERSION = 1

__all__ = ["SCHEMA_VERSION", "SceneFormatError", "render_scene", "parse_scene", "save_scene", "load_scene"]


class SceneFormatError(ValueError):
    """A scene document that cannot be accepted, with the offending path (sceneio.py:23-28)."""

    def __init__(self, path: str, message: str):
        self.path = path
        super().__init__(f"{path}: {message}")


def _vec(a) -> list:
    return [float(c) for c in a]


def render_scene(scene) -> str:
    """Serialize ``scene`` (Scene, ArrayScene or a reference Scene) to the
    versioned document text (sceneio.py:57-75).  The masses and springs
    arrays are written by the native codec (csrc/sceneio.cpp) around the rest
    of the document, which json.dumps renders; non-finite values go through
    the host writer, which raises the reference's error."""
    native = _render_native(scene)
    if native is None:
        return _render_host(scene)
    ptr, n = native
    return _take_text(ptr, n)


def _small_doc(scene, a, masses, springs) -> dict:
    labels = [g[0] for g in a.group_params]
    mats = [{"name": mt.name, "k0": mt.k0, "l_ref": mt.l_ref, "density": mt.density,
             "total_mass": mt.total_mass, "mass_per_node": mt.mass_per_node}
            for mt in getattr(scene, "materials", [])]
    groups = [{"label": lab, "mode": mode, "amplitude": amp, "frequency": freq, "phase": ph}
              for lab, mode, amp, freq, ph in a.group_params]
    planes = [{"normal": _vec(nrm), "offset": off, "penalty": pen, "friction": fr}
              for nrm, off, pen, fr in a.planes]
    return {"schema_version": SCHEMA_VERSION, "gravity": _vec(a.gravity), "dt": a.dt, "damping": a.damping,
            "masses": masses, "springs": springs, "materials": mats, "groups": groups, "planes": planes}, labels


def _dumps(doc) -> str:
    try:
        return json.dumps(doc, indent=2, allow_nan=False) + "\n"
    except ValueError as exc:
        raise SceneFormatError("$", f"non-finite value in scene: {exc}") from exc


def _render_host(scene) -> str:
    a = scene_arrays(scene)
    doc, labels = _small_doc(scene, a, None, None)
    doc["masses"], doc["springs"] = _mass_entries(a), _spring_entries(a, labels)
    return _dumps(doc)


def _render_native(scene):
    """(pointer, length) of the whole document rendered natively (free with
    ss_doc_free_text), or None when a value is non-finite."""
    a = scene_arrays(scene)
    doc, labels = _small_doc(scene, a, [], [])
    text = _dumps(doc)                       # the small values; raises on non-finite ones
    nm, ns = a.m.shape[0], a.si.shape[0]
    im = text.index('\n  "masses": [],\n') + 3
    js = text.index('\n  "springs": [],\n') + 3
    pre = text[:im] + ('"masses": [\n' if nm else '"masses": []')
    mid = ("\n  ]" if nm else "") + text[im + len('"masses": []'):js] + ('"springs": [\n' if ns else '"springs": []')
    post = ("\n  ]" if ns else "") + text[js + len('"springs": []'):]
    lib = _lib.lib()
    f64 = lambda arr: np.ascontiguousarray(arr, dtype=np.float64)
    m, x, v, f = f64(a.m), f64(a.x), f64(a.v), f64(a.f_ext)
    fixed = np.ascontiguousarray(a.fixed, dtype=np.uint8)
    si = np.ascontiguousarray(a.si, dtype=np.int64)
    sj = np.ascontiguousarray(a.sj, dtype=np.int64)
    k, l0 = f64(a.k), f64(a.l0)
    group = None if a.group is None else np.ascontiguousarray(a.group, dtype=np.int32)
    lab = (C.c_char_p * max(1, len(labels)))(*[json.dumps(t).encode("ascii") for t in labels])
    ptr, n = C.c_void_p(), C.c_int64()
    rc = lib.ss_doc_render(nm, _lib.dptr(m), _lib.dptr(x), _lib.dptr(v), _lib.dptr(f), _lib.u8ptr(fixed),
                           ns, _lib.i64ptr(si), _lib.i64ptr(sj), _lib.dptr(k), _lib.dptr(l0), _lib.i32ptr(group),
                           lab, len(labels), pre.encode("ascii"), mid.encode("ascii"), post.encode("ascii"),
                           C.byref(ptr), C.byref(n))
    if rc == _lib.SS_EFALLBACK:
        return None
    _lib.check(rc, "ss_doc_render")
    return ptr, n.value


def _mass_entries(a) -> list:
    x, v, f = a.x.tolist(), a.v.tolist(), a.f_ext.tolist()
    m, fixed = a.m.tolist(), a.fixed.tolist()
    return [{"id": i, "m": m[i], "x": x[i], "v": v[i], "f_ext": f[i], "fixed": bool(fixed[i])}
            for i in range(len(m))]


def _spring_entries(a, labels) -> list:
    si, sj, k, l0 = a.si.tolist(), a.sj.tolist(), a.k.tolist(), a.l0.tolist()
    grp = a.group.tolist() if a.group is not None else None
    return [{"id": s, "i": si[s], "j": sj[s], "k": k[s], "l0": l0[s],
             "group": (labels[grp[s]] if grp is not None and grp[s] >= 0 else None)}
            for s in range(len(si))]


def _take_text(ptr, n) -> str:
    lib = _lib.lib()
    try:
        return C.string_at(ptr, n).decode("ascii")
    finally:
        lib.ss_doc_free_text(ptr)


# ------------------------------------------------------------ parsing

def _is_number(value) -> bool:
    return isinstance(value, (int, float)) and not isinstance(value, bool)


def _named(what: str):
    return lambda value: f"expected {what}, got {type(value).__name__}"


def _same(value):
    return value


# kind -> (accepts?, conversion, complaint) -- the field types of the
# reference's document schema (sceneio.py:98-136)
_KINDS = {
    "number": (_is_number, float, _named("a number")),
    "number?": (lambda v: v is None or _is_number(v), lambda v: None if v is None else float(v), _named("a number")),
    "int": (lambda v: isinstance(v, int) and not isinstance(v, bool), _same, _named("an integer")),
    "bool": (lambda v: isinstance(v, bool), _same, _named("a boolean")),
    "string": (lambda v: isinstance(v, str), _same, _named("a string")),
    "string?": (lambda v: v is None or isinstance(v, str), _same, _named("a string or null")),
    "vec3": (lambda v: isinstance(v, list) and len(v) == 3 and all(map(_is_number, v)),
             lambda v: tuple(map(float, v)), lambda v: "expected a list of three numbers"),
    "list": (lambda v: isinstance(v, list), _same, _named("a list")),
}


def _coerce(value, path: str, kind):
    """``value`` checked against and converted to ``kind``, else SceneFormatError at ``path``."""
    accepts, convert, complaint = _KINDS[kind]
    if not accepts(value):
        raise SceneFormatError(path, complaint(value))
    return convert(value)


def _expect(obj, path: str, required: dict, optional: dict) -> dict:
    """The fields of a JSON object: no unknown keys (first one in document
    order is reported), every required key present, each value of its kind;
    absent optional keys take their defaults."""
    if not isinstance(obj, dict):
        raise SceneFormatError(path, _named("an object")(obj))
    stray = next((key for key in obj if key not in required and key not in optional), None)
    if stray is not None:
        raise SceneFormatError(f"{path}.{stray}", "unknown field")
    missing = next((key for key in required if key not in obj), None)
    if missing is not None:
        raise SceneFormatError(path, f"missing required field {missing!r}")
    fields = {key: _coerce(obj[key], f"{path}.{key}", kind) for key, kind in required.items()}
    fields.update((key, _coerce(obj[key], f"{path}.{key}", kind) if key in obj else default)
                  for key, (kind, default) in optional.items())
    return fields


_TOP = dict(required={"schema_version": "int", "gravity": "vec3", "dt": "number", "masses": "list",
                      "springs": "list"},
            optional={"damping": ("number", 0.0), "materials": ("list", []), "groups": ("list", []),
                      "planes": ("list", [])})
_MASS = dict(required={"m": "number", "x": "vec3"},
             optional={"id": ("int", None), "v": ("vec3", (0.0, 0.0, 0.0)), "f_ext": ("vec3", (0.0, 0.0, 0.0)),
                       "fixed": ("bool", False)})
_SPRING = dict(required={"i": "int", "j": "int", "k": "number", "l0": "number"},
               optional={"id": ("int", None), "group": ("string?", None)})
_MATERIAL = dict(required={"name": "string"},
                 optional={"k0": ("number", 10000.0), "l_ref": ("number?", None), "density": ("number?", None),
                           "total_mass": ("number?", None), "mass_per_node": ("number?", None)})
_GROUP = dict(required={"label": "string", "mode": "string"},
              optional={"amplitude": ("number", 0.0), "frequency": ("number", 1.0), "phase": ("number", 0.0)})
_PLANE = dict(required={"normal": "vec3"},
              optional={"offset": ("number", 0.0), "penalty": ("number", 1e5), "friction": ("number", 0.0)})


def parse_scene(text: str) -> ArrayScene:
    """Parse and validate a scene document (sceneio.py:173-239) into arrays.
    The native fast path (csrc/sceneio.cpp) decodes plain documents; any
    document it does not accept whole goes through the host parser below,
    which reports the reference's error for it."""
    fast = _parse_native(text)
    return fast if fast is not None else _parse_host(text)


def _check_top(raw) -> dict:
    top = _expect(raw, "$", **_TOP)
    if top["schema_version"] != SCHEMA_VERSION:
        raise SceneFormatError("$.schema_version",
                               f"unsupported version {top['schema_version']} (this reader handles {SCHEMA_VERSION})")
    return top


def _parse_native(text: str):
    if not text.isascii():
        return None
    return _parse_native_bytes(text.encode("ascii"))


def _parse_native_bytes(raw_bytes: bytes):
    lib = _lib.lib()
    h = C.c_void_p()
    rc = lib.ss_doc_parse(raw_bytes, len(raw_bytes), C.byref(h))
    if rc == _lib.SS_EFALLBACK:
        return None
    _lib.check(rc, "ss_doc_parse")
    try:
        nm, ns = C.c_int64(), C.c_int64()
        nk, nl = C.c_int32(), C.c_int32()
        _lib.check(lib.ss_doc_info(h, C.byref(nm), C.byref(ns), C.byref(nk), C.byref(nl)), "ss_doc_info")
        raw = {}
        for i in range(nk.value):
            name, off, span = C.c_char_p(), C.c_int64(), C.c_int64()
            _lib.check(lib.ss_doc_key(h, i, C.byref(name), C.byref(off), C.byref(span)), "ss_doc_key")
            key = name.value.decode("ascii")
            raw[key] = [] if key in ("masses", "springs") else json.loads(raw_bytes[off.value:off.value + span.value])
        top = _check_top(raw)
        n, s = nm.value, ns.value
        m, x, v, f = np.empty(n), np.empty((n, 3)), np.empty((n, 3)), np.empty((n, 3))
        fixed = np.empty(n, dtype=np.uint8)
        _lib.check(lib.ss_doc_masses(h, _lib.dptr(m), _lib.dptr(x), _lib.dptr(v), _lib.dptr(f), _lib.u8ptr(fixed)),
                   "ss_doc_masses")
        si, sj = np.empty(s, dtype=np.int64), np.empty(s, dtype=np.int64)
        k, l0 = np.empty(s), np.empty(s)
        lab = np.empty(s, dtype=np.int32)
        _lib.check(lib.ss_doc_springs(h, _lib.i64ptr(si), _lib.i64ptr(sj), _lib.dptr(k), _lib.dptr(l0),
                                      _lib.i32ptr(lab)), "ss_doc_springs")
        names = [lib.ss_doc_label(h, g).decode("ascii") for g in range(nl.value)]
    finally:
        lib.ss_doc_free(h)
    dup = _first_duplicate(si, sj, n)       # every entry decoded cleanly: the first duplicate is the first error
    if dup is not None:
        raise SceneFormatError(f"$.springs[{dup}]", f"duplicate spring between masses {si[dup]} and {sj[dup]}")
    return _assemble(top, x, v, f, m, fixed.astype(bool), si, sj, k, l0, names, lab)


def _parse_host(text: str) -> ArrayScene:
    try:
        raw = json.loads(text)
    except json.JSONDecodeError as exc:
        raise SceneFormatError("$", f"malformed document: {exc}") from exc
    top = _check_top(raw)
    n = len(top["masses"])
    x = np.empty((n, 3))
    v = np.empty((n, 3))
    f = np.empty((n, 3))
    m = np.empty(n)
    fixed = np.zeros(n, dtype=bool)
    for idx, entry in enumerate(top["masses"]):
        path = f"$.masses[{idx}]"
        fl = _expect(entry, path, **_MASS)
        if fl["id"] is not None and fl["id"] != idx:
            raise SceneFormatError(f"{path}.id", f"ids must be contiguous; expected {idx}")
        x[idx], v[idx], f[idx], m[idx], fixed[idx] = fl["x"], fl["v"], fl["f_ext"], fl["m"], fl["fixed"]
    s_count = len(top["springs"])
    si = np.empty(s_count, dtype=np.int64)
    sj = np.empty(s_count, dtype=np.int64)
    k = np.empty(s_count)
    l0 = np.empty(s_count)
    names: list = []
    lab = np.full(s_count, -1, dtype=np.int32)
    pairs = set()
    for idx, entry in enumerate(top["springs"]):
        path = f"$.springs[{idx}]"
        fl = _expect(entry, path, **_SPRING)
        if fl["id"] is not None and fl["id"] != idx:
            raise SceneFormatError(f"{path}.id", f"ids must be contiguous; expected {idx}")
        for end in ("i", "j"):
            if not 0 <= fl[end] < n:
                raise SceneFormatError(f"{path}.{end}", f"no such mass {fl[end]}")
        pair = (min(fl["i"], fl["j"]), max(fl["i"], fl["j"]))
        if pair in pairs:                   # Scene.add_spring (model.py:171-176) raises inside the loop
            raise SceneFormatError(path, f"duplicate spring between masses {fl['i']} and {fl['j']}")
        pairs.add(pair)
        si[idx], sj[idx], k[idx], l0[idx] = fl["i"], fl["j"], fl["k"], fl["l0"]
        if fl["group"] is not None:
            if fl["group"] not in names:
                names.append(fl["group"])
            lab[idx] = names.index(fl["group"])
    return _assemble(top, x, v, f, m, fixed, si, sj, k, l0, names, lab)


def _assemble(top, x, v, f, m, fixed, si, sj, k, l0, names, lab) -> ArrayScene:
    """Materials, groups, planes and the whole-scene checks (sceneio.py:
    210-239) over decoded columns; ``lab`` indexes ``names``, the distinct
    spring group strings (-1: no group)."""
    s_count = si.shape[0]
    mats = [Material(**_expect(e, f"$.materials[{i}]", **_MATERIAL)) for i, e in enumerate(top["materials"])]
    groups = {}
    for i, e in enumerate(top["groups"]):
        fl = _expect(e, f"$.groups[{i}]", **_GROUP)
        try:
            g = ActuationGroup(**fl)
        except ValueError as exc:
            raise SceneFormatError(f"$.groups[{i}]", str(exc)) from exc
        if g.label in groups:
            raise SceneFormatError(f"$.groups[{i}]", f"duplicate actuation group {g.label!r}")
        groups[g.label] = g
    labels = list(groups)
    group = None
    unknown = [t for t in names if t not in groups]
    if (lab >= 0).any():                    # defined labels -> group index; others -> -2 - q (validate_scene reports them)
        lut = np.array([labels.index(t) if t in groups else -2 - unknown.index(t) for t in names], dtype=np.int32)
        group = np.where(lab >= 0, lut[np.maximum(lab, 0)], -1).astype(np.int32)
    planes = [ContactPlane(**_expect(e, f"$.planes[{i}]", **_PLANE)) for i, e in enumerate(top["planes"])]
    scene = ArrayScene(x=x, m=m, si=si, sj=sj, k=k, l0=l0, v=v, f_ext=f, fixed=fixed, gravity=top["gravity"],
                       dt=top["dt"], damping=top["damping"], groups=groups, group=None, planes=planes,
                       materials=mats)
    if group is not None:
        scene.group = group
        scene.unknown_group_labels = unknown
    violations = validate_scene(scene)
    if violations:
        first = violations[0]
        raise SceneFormatError(f"$.{first.where}", first.message)
    return scene


def _first_duplicate(si, sj, n):
    """Lowest spring index whose unordered pair occurred before (Scene.add_spring's
    duplicate rule, model.py:171-176), or None: one stable sort of pair keys."""
    if si.shape[0] < 2:
        return None
    lo, hi = np.minimum(si, sj), np.maximum(si, sj)
    key = lo * max(int(n), 1) + hi
    order = np.argsort(key, kind="stable")
    k = key[order]
    repeat = k[1:] == k[:-1]
    return int(order[1:][repeat].min()) if repeat.any() else None


def save_scene(scene, path) -> None:
    """Write the document; the natively rendered text goes to the file
    straight from the library's buffer."""
    native = _render_native(scene)
    if native is None:
        with open(path, "w") as fh:
            fh.write(_render_host(scene))
        return
    ptr, n = native
    try:
        with open(path, "wb") as fh:
            fh.write(memoryview((C.c_char * n).from_address(ptr.value)) if n else b"")
    finally:
        _lib.lib().ss_doc_free_text(ptr)


def load_scene(path) -> ArrayScene:
    """Read and parse a document: the native fast path reads the file's bytes
    as they are; anything it does not accept is parsed from the text."""
    with open(path, "rb") as fh:
        raw = fh.read()
    fast = _parse_native_bytes(raw) if raw.isascii() else None
    if fast is not None:
        return fast
    return _parse_host(raw.decode("utf-8"))
