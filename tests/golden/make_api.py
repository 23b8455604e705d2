"""Record the reference's public API surface (names + call signatures) as a fixture.

    python tests/golden/make_api.py      # build container only (/root/reference)

tests/test_api_surface.py checks the drop-in facade against tests/golden/api.json
on any machine (the GPU box has no reference).
"""

import inspect
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
import linksdf as ref  # noqa: E402  (reference, read-only)

out = {}
for name in sorted(n for n in dir(ref) if not n.startswith("_")):
    obj = getattr(ref, name)
    if inspect.ismodule(obj):
        out[name] = {"kind": "module"}
        continue
    entry = {"kind": "class" if inspect.isclass(obj) else "function"}
    target = obj.__init__ if inspect.isclass(obj) else obj
    try:
        sig = inspect.signature(target)
        entry["params"] = [[p.name, p.kind.name, p.default is not inspect.Parameter.empty]
                           for p in sig.parameters.values() if p.name != "self"]
    except (TypeError, ValueError):
        pass
    if inspect.isclass(obj):
        entry["methods"] = sorted(m for m in vars(obj) if not m.startswith("_"))
    out[name] = entry
(Path(__file__).resolve().parent / "api.json").write_text(json.dumps(out, indent=1, sort_keys=True))
print(len(out), "names")
