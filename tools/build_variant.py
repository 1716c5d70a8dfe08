"""Build an experimental variant of libklnmf.so with extra nvcc defines
(e.g. the long-row CTA shape) into _variants/<name>/libklnmf.so; select it
at run time with KLNMF_LIB=_variants/<name>/libklnmf.so.

    python tools/build_variant.py cl128 -DKLNMF_CL_NT=128 -DKLNMF_CL_PER_SM=4
"""
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
from paper_1604_04026_b200 import build as kb  # noqa: E402


def main():
    name, defines = sys.argv[1], sys.argv[2:]
    # "--src FILE": compile another solve_fast.cu (e.g. an older revision's)
    src_fast = kb.CSRC / "solve_fast.cu"
    if "--src" in defines:
        i = defines.index("--src")
        src_fast = Path(defines[i + 1]).resolve()
        defines = defines[:i] + defines[i + 2:]
    out = REPO / "_variants" / name
    out.mkdir(parents=True, exist_ok=True)
    lib = kb.build()  # the regular objects are reused for every other file
    objs = []
    for src in kb.SOURCES:
        if src == "solve_fast.cu":
            o = out / "solve_fast.o"
            subprocess.run([kb.nvcc(), *kb.ARCH, *kb.COMMON, "-I", str(kb.CSRC), *defines, "-c", str(src_fast),
                            "-o", str(o)], check=True)
        else:
            o = kb.OBJDIR / (Path(src).stem + ".o")
        objs.append(str(o))
    subprocess.run([kb.nvcc(), *kb.ARCH, "-shared", "-Xcompiler", "-pthread", "-o", str(out / "libklnmf.so"),
                    *objs], check=True)
    print(out / "libklnmf.so", "(base", lib, ")")


if __name__ == "__main__":
    main()
