"""parse_scene on 148 mutated documents against the reference's outcome for
the same text (tests/golden/scene_errors.json, made by
tests/golden/make_scene_errors.py with the unmodified reference): the same
error path and message, or a scene rendering to the same bytes.  Both the
native fast path and the host parser are exercised."""
import hashlib
import json
import os

import pytest

from paper_2207_09334_b200 import sceneio as S

from scene_mutations import documents

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scene_errors.json")))
DOCS = documents()


def outcome(fn, text):
    try:
        return ["ok", hashlib.sha256(S.render_scene(fn(text)).encode()).hexdigest()]
    except S.SceneFormatError as exc:
        return ["error", exc.path, str(exc)]


def test_fixture_covers_every_document():
    assert sorted(GOLD) == sorted(name for name, _ in DOCS)


@pytest.mark.parametrize("name,text", DOCS, ids=[n for n, _ in DOCS])
def test_same_outcome_as_the_reference(name, text):
    assert outcome(S.parse_scene, text) == GOLD[name]
    assert outcome(S._parse_host, text) == GOLD[name]
