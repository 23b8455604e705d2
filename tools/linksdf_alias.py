"""pytest plugin: ``import linksdf`` (the reference package) resolves to this
package, so the reference's own test modules run against the drop-in facade.

    python -m pytest <reference tests> -p linksdf_alias      (tools/ on sys.path)

Used by tools/reference_tests.py; nothing here is on the product path.
"""
import importlib
import sys

import paper_2309_12543_b200 as _pkg

sys.modules["linksdf"] = _pkg
for _sub in ("approx", "errors", "grids", "meshes", "placement", "query", "robot", "checker", "replay"):
    sys.modules[f"linksdf.{_sub}"] = importlib.import_module(f"paper_2309_12543_b200.{_sub}")
