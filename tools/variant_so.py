"""Build a variant of libsgtr.so for an A/B timing run (not product code).

  python tools/variant_so.py NAME FILE 'OLD=>NEW' ['OLD=>NEW' ...]

compiles csrc/FILE with each literal OLD replaced by NEW (each must occur),
links it with the other objects of the current build and writes
_variants/NAME.so; run the bench against it with SGTR_LIB=_variants/NAME.so.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2602_00395_b200"))
import build as B  # noqa: E402


def main():
    name, src, subs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    text = open(os.path.join(B.CSRC, src)).read()
    for sub in subs:
        old, new = sub.split("=>", 1)
        if old not in text:
            raise SystemExit(f"{old!r} not found in {src}")
        text = text.replace(old, new)
    out_dir = os.path.join(ROOT, "_variants")
    os.makedirs(out_dir, exist_ok=True)
    tmp_src = os.path.join(B.CSRC, f"_variant_{name}_{src}")
    open(tmp_src, "w").write(text)
    obj = os.path.join(out_dir, f"{name}_{src}.o")
    try:
        cmd = [B.NVCC] + B.COMMON + (["--fmad=false"] if src in B.NO_FMA else []) + \
            ["-c", tmp_src, "-o", obj, "-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
    finally:
        os.remove(tmp_src)
    objs = [obj if s == src else os.path.join(B.OBJ, s.replace(".cu", ".o")) for s in B.SOURCES]
    lib = os.path.join(out_dir, f"{name}.so")
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs + ["-ldl", "-lpthread"],
                   check=True)
    print(lib)


if __name__ == "__main__":
    main()
