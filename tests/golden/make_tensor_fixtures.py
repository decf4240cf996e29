"""LPATTN-TENSOR v1 regression fixture made by the UNMODIFIED reference.

    python tests/golden/make_tensor_fixtures.py [/root/reference/pkg/src]

Mirrors the reference CLI's file workflow (cli.py:130-141 `gen`, cli.py:145-176 + 211-222 `run`):
Q/K/V are drawn by the reference's `tensorio.generate` (Philox, gaussian, seeds s, s+1, s+2) and
written with its `tensorio.write_tensor` (+ JSON sidecars); `attention_quantized` runs on them and
its output is written as a fourth tensor file, its run report (the CLI's `run` row without the
wall time) as run.json.  The GPU test reads the files with paper_2505_21136_b200.tensorio.load.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent / "lpattn_tensor"
REF_SRC = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))

from lpattn import tensorio  # noqa: E402
from lpattn.attention import AttentionConfig, attention_quantized, attention_reference  # noqa: E402
from lpattn.metrics import compare  # noqa: E402

HEADS, SEQ, DIM, SEED = 2, 200, 64, 21


def main() -> None:
    HERE.mkdir(exist_ok=True)
    shape = (HEADS, SEQ, DIM)
    arrs = {}
    for name, off in (("q", 0), ("k", 1), ("v", 2)):
        arr, meta = tensorio.generate(shape, "gaussian", SEED + off)
        tensorio.write_tensor(HERE / f"{name}.bin", arr, meta)
        arrs[name] = tensorio.read_tensor(HERE / f"{name}.bin")  # float32, as the CLI reads it
    cfg = AttentionConfig(seq_len=SEQ, head_dim=DIM, num_heads=HEADS)
    report = attention_quantized(arrs["q"], arrs["k"], arrs["v"], cfg)
    exact = attention_reference(arrs["q"], arrs["k"], arrs["v"], cfg)
    m = compare(exact, report.output)
    tensorio.write_tensor(HERE / "out.bin", report.output, {"producer": "lpattn.attention_quantized"})
    row = {"heads": HEADS, "seq_len": SEQ, "head_dim": DIM, "seed": SEED, "cossim": m.cossim, "l1": m.l1,
           "rmse": m.rmse, "overflow_events": report.overflow_events,
           "fp16_to_fp32_conversions": report.fp16_to_fp32_conversions,
           "mma_invocations": report.mma_invocations}
    (HERE / "run.json").write_text(json.dumps(row, indent=2, sort_keys=True) + "\n")
    print(json.dumps(row))


if __name__ == "__main__":
    main()
