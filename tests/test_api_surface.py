"""The drop-in boundary: the facade exposes every public name
of the reference package with call signatures the reference's callers can use
unchanged.  The reference surface is pinned in tests/golden/api.json
(tests/golden/make_api.py, generated from /root/reference in the build
container).  CPU only: no kernel runs here.
"""

import inspect
import json
from pathlib import Path

import pytest

import paper_2309_12543_b200 as L

API = json.loads((Path(__file__).resolve().parent / "golden" / "api.json").read_text())


@pytest.mark.parametrize("name", sorted(API))
def test_name_exported_with_compatible_signature(name):
    entry = API[name]
    assert hasattr(L, name), f"{name} missing from the facade"
    obj = getattr(L, name)
    if entry["kind"] == "module":
        assert inspect.ismodule(obj)
        return
    if entry["kind"] == "class":
        assert inspect.isclass(obj)
        missing = [m for m in entry.get("methods", []) if not hasattr(obj, m)]
        assert not missing, f"{name} lacks {missing}"
    if "params" not in entry:
        return
    target = obj.__init__ if inspect.isclass(obj) else obj
    ours = [p for p in inspect.signature(target).parameters.values() if p.name != "self"]
    ref = entry["params"]
    # the reference's parameters, in order, with the same kinds ...
    assert [(p.name, p.kind.name) for p in ours[:len(ref)]] == [(n, k) for n, k, _ in ref], name
    # ... where the reference has a default we have one too, and anything we add is optional
    for p, (_, _, has_default) in zip(ours, ref):
        if has_default:
            assert p.default is not inspect.Parameter.empty, f"{name}.{p.name} lost its default"
    for p in ours[len(ref):]:
        assert p.default is not inspect.Parameter.empty or p.kind in (p.VAR_POSITIONAL, p.VAR_KEYWORD), \
            f"{name} adds a required parameter {p.name}"


def test_query_has_no_pose_or_rotation_parameter():
    """Acceptance C7 (test_acceptance.py:389-391): the query takes no poses or rotations."""
    for p in inspect.signature(L.query_min_distances).parameters:
        assert "pose" not in p and "rotation" not in p


def test_additions_are_keyword_only_or_new_names():
    sig = inspect.signature(L.query_min_distances)
    assert sig.parameters["return_argmin"].kind is inspect.Parameter.KEYWORD_ONLY
    for extra in ("TrajectorySdf", "query_trajectory", "DistanceChecker", "CheckerPipeline"):
        assert hasattr(L, extra) and extra not in API
