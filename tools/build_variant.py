"""Build an A/B variant of the library: lsdf_query.cu recompiled with extra
nvcc defines, linked with the other objects of the current build.

    python tools/build_variant.py OUT.so -DLSDF_SHELL_MINB=4
    python tools/build_variant.py OUT.so --src old_query.cu   (e.g. from `git show HEAD~1:...`)
    python tools/build_variant.py OUT.so --unit lsdf_voxel.cu --src old_voxel.cu

Select it at run time with LINKSDF_B200_LIB=OUT.so (paper_2309_12543_b200/_native.py).
"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2309_12543_b200 import build as B  # noqa: E402


def main(out, args, source="lsdf_query.cu"):
    B.build()
    nvcc = B._nvcc()
    if "--unit" in args:  # which translation unit the variant replaces (default lsdf_query.cu)
        k = args.index("--unit")
        source = args[k + 1]
        args = args[:k] + args[k + 2:]
    src = B.CSRC / source
    if "--src" in args:  # another version of lsdf_query.cu (compiled from the csrc directory for its includes)
        k = args.index("--src")
        src = B.CSRC / ("_variant_" + Path(args[k + 1]).name)
        src.write_text(Path(args[k + 1]).read_text())
        args = args[:k] + args[k + 2:]
    defines = args
    obj = B.OUT_DIR / (Path(source).stem + ".variant.o")
    cmd = [nvcc, *B.ARCH, *B.FLAGS, *defines, "-I", str(B.INCLUDE), "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if src.name.startswith("_variant_"):
        src.unlink()
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
