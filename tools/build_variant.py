"""Build a variant of libvsb200.so with extra nvcc defines into variants/lib_<name>.so (dev
tuning; run the variants with VSB200_LIB=... e.g. through tools/tune_variants.sh).
usage: build_variant.py NAME [-DFOO=1 ...]"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1912_09596_b200 import _build  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = _build.ROOT / "variants"
out.mkdir(exist_ok=True)
objdir = out / f"obj_{name}"
objdir.mkdir(exist_ok=True)
procs, objs = [], []
import os  # noqa: E402
srcdir = os.environ.get("VARIANT_SRC")  # optional: another csrc tree (e.g. a git checkout)
sources = sorted(Path(srcdir).glob("*.cu")) if srcdir else _build.sources()
for src in sources:
    obj = objdir / (src.stem + ".o")
    cmd = [_build._nvcc(), *_build.NVCC_FLAGS, *extra, "-I", str(_build.ROOT / "include"), "-c",
           str(src), "-o", str(obj)]
    procs.append(subprocess.Popen(cmd))
    objs.append(str(obj))
if any(p.wait() for p in procs):
    sys.exit("nvcc failed")
subprocess.run([_build._nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                "-o", str(out / f"lib_{name}.so"), "-lcudart_static", "-lrt", "-lpthread", "-ldl"],
               check=True)
print(out / f"lib_{name}.so")
