"""Run the reference's own test suite against the facade.

    python tools/reference_tests.py stage   # build container: copy /root/reference/pkg/tests
                                            #   into baseline/_ref/tests (git-ignored, travels to the GPU box)
    python tools/reference_tests.py run     # GPU box: pytest those modules with `linksdf` aliased to
                                            #   paper_2309_12543_b200 (tools/linksdf_alias.py)

The staged copy is test input only: it is not in the repository's history and
no product code reads it.  The run writes a per-test outcome list and a
summary to gpurun_out/reference_tests.txt.
"""
import os
import shutil
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
STAGE = REPO / "baseline" / "_ref" / "tests"
SRC = Path("/root/reference/pkg/tests")


def stage():
    if STAGE.exists():
        shutil.rmtree(STAGE)
    STAGE.mkdir(parents=True)
    for f in sorted(SRC.glob("*.py")):
        shutil.copy2(f, STAGE / f.name)
    print(f"staged {len(list(STAGE.glob('*.py')))} files into {STAGE}")


def run():
    out = REPO / "gpurun_out" / "reference_tests.txt"
    out.parent.mkdir(exist_ok=True)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REPO / "tools"), str(REPO)]))
    cmd = [sys.executable, "-m", "pytest", str(STAGE), "-p", "linksdf_alias", "-p", "no:cacheprovider",
           "--rootdir", str(STAGE), "--continue-on-collection-errors", "-q", "-rA", "--tb=line", "-o", "console_output_style=classic"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=str(STAGE))
    out.write_text(r.stdout[-200_000:] + "\n---- stderr ----\n" + r.stderr[-20_000:])
    print(r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:])


if __name__ == "__main__":
    {"stage": stage, "run": run}[sys.argv[1]]()
