"""Outcome of the REFERENCE's sceneio.parse_scene on every mutated document
of tests/scene_mutations.py: ("ok", render of the parsed scene's sha256) or
("error", path, message) -> tests/golden/scene_errors.json.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_scene_errors.py
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from springsim.sceneio import SceneFormatError, parse_scene, render_scene  # noqa: E402

from scene_mutations import documents  # noqa: E402

if __name__ == "__main__":
    out = {}
    for name, text in documents():
        try:
            sc = parse_scene(text)
            out[name] = ["ok", hashlib.sha256(render_scene(sc).encode()).hexdigest()]
        except SceneFormatError as exc:
            out[name] = ["error", exc.path, str(exc)]
    with open(os.path.join(HERE, "scene_errors.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(len(out), "documents,", sum(v[0] == "error" for v in out.values()), "errors")
