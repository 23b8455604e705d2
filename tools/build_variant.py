"""Build an A/B variant of the library: lsdf_query.cu recompiled with extra
nvcc defines, linked with the other objects of the current build.

    python tools/build_variant.py OUT.so -DLSDF_SHELL_MINB=4 -DLSDF_SLIM_SETUP=1

Select it at run time with LINKSDF_B200_LIB=OUT.so (paper_2309_12543_b200/_native.py).
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_12543_b200 import build as B  # noqa: E402


def main(out, defines, source="lsdf_query.cu"):
    B.build()
    nvcc = B._nvcc()
    obj = B.OUT_DIR / (Path(source).stem + ".variant.o")
    cmd = [nvcc, *B.ARCH, *B.FLAGS, *defines, "-I", str(B.INCLUDE), "-c", str(B.CSRC / source), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.exit(r.stdout + r.stderr)
    log = [ln for ln in (r.stdout + r.stderr).splitlines() if "registers" in ln or "spill" in ln]
    objs = [str(obj) if Path(n).stem == Path(source).stem else str(B.OUT_DIR / (Path(n).stem + ".o"))
            for n in B.SOURCES]
    subprocess.run([nvcc, *B.ARCH, "-shared", "-o", out, *objs, "-lcuda"], check=True)
    obj.unlink()
    print("\n".join(log[:16]))
    print("built", out)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
