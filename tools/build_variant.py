"""Build an A/B variant of libsa2pp.so with -D overrides on one source (development aid).

    python tools/build_variant.py NAME attn_ws.cu -DSA2PP_WS_REG_SOFTMAX=96 ...
writes variants/libsa2pp_NAME.so (git-ignored, travels to the GPU box); select it with SA2PP_LIB.
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2505_21136_b200 import build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
out = ROOT / "variants"
out.mkdir(exist_ok=True)
obj = out / f"{Path(src).stem}_{name}.o"
subprocess.run([B.nvcc(), *B.ARCH, *B.FLAGS, *defs, "-c", str(B.CSRC / src), "-o", str(obj)], check=True)
objs = [str(obj) if Path(s).stem == Path(src).stem else str(B.BUILD / (Path(s).stem + ".o")) for s in B.SOURCES]
lib = out / f"libsa2pp_{name}.so"
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", str(lib)], check=True)
print(lib)
