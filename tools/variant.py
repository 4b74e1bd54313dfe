"""Build an experiment variant of libiga with extra nvcc defines (A/B timing on the GPU box).

    python tools/variant.py NAME "-DFOO=1 ..."   ->  scratch/libiga_NAME.so  (scratch/ is git-ignored
                                                    but travels to the GPU box with gpurun)
Load it with IGA_LIB=$PWD/scratch/libiga_NAME.so (see tools/ab.sh)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["IGA_NVCC_EXTRA"] = sys.argv[2] if len(sys.argv) > 2 else ""
import paper_1305_4452_b200.build as b  # noqa: E402  (reads IGA_NVCC_EXTRA at import)

name = sys.argv[1]
b.BUILD = os.path.join(ROOT, "scratch", "build_" + name)
b.SO = os.path.join(ROOT, "scratch", "libiga_" + name + ".so")
b.build(force=True)
print(b.SO)
