"""LPATTN-TENSOR v1 container (paper_2505_21136_b200/tensorio.py), SURVEY §8(f3)."""

import numpy as np
import pytest
import torch

from paper_2505_21136_b200 import tensorio as tio


def test_roundtrip_bytes_and_values(tmp_path):
    x = np.random.default_rng(0).normal(size=(2, 3, 5)).astype(np.float32)
    p = tmp_path / "x.bin"
    tio.write_tensor(p, x, {"seed": 0})
    assert np.array_equal(tio.read_tensor(p), x)
    raw = p.read_bytes()
    assert raw[:16] == tio.MAGIC and len(raw) == 16 + 8 * 5 + 4 * x.size
    assert (tmp_path / "x.bin.meta.json").exists()
    t = tio.load(p, device="cpu")
    assert torch.equal(t, torch.from_numpy(x))


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"X" + b[1:], "bad magic"),
    (lambda b: b[:16] + (2).to_bytes(8, "little") + b[24:], "unsupported version"),
    (lambda b: b[:-4], "truncated payload"),
    (lambda b: b + b"\0", "trailing bytes"),
])
def test_rejects_malformed(tmp_path, mutate, msg):
    p = tmp_path / "x.bin"
    tio.write_tensor(p, np.ones((2, 2), np.float32))
    p.write_bytes(mutate(p.read_bytes()))
    with pytest.raises(tio.TensorFormatError, match=msg):
        tio.read_tensor(p)


def test_interchangeable_with_reference(lpattn, tmp_path):
    from lpattn import tensorio as ref
    x, meta = ref.generate((3, 7, 4), "gaussian", 5)
    ref.write_tensor(tmp_path / "r.bin", x, meta)
    tio.write_tensor(tmp_path / "o.bin", x)
    assert (tmp_path / "r.bin").read_bytes() == (tmp_path / "o.bin").read_bytes()
    assert np.array_equal(ref.read_tensor(tmp_path / "o.bin"), tio.read_tensor(tmp_path / "r.bin"))


FIX = __import__("pathlib").Path(__file__).resolve().parent / "golden" / "lpattn_tensor"


def test_reference_tensor_fixture_oracle_parity():
    """The LPATTN-TENSOR fixture written by the unmodified reference (tests/golden/make_tensor_fixtures.py)
    reads back through this reader and the oracle reproduces the reference's output file and run row."""
    import json

    from oracle import sage_cpu as oc
    q, k, v = (tio.read_tensor(FIX / f"{n}.bin") for n in ("q", "k", "v"))
    ref_out = tio.read_tensor(FIX / "out.bin")
    row = json.loads((FIX / "run.json").read_text())
    cfg = oc.AttentionConfig(seq_len=row["seq_len"], head_dim=row["head_dim"], num_heads=row["heads"])
    rep = oc.attention_quantized(q, k, v, cfg)
    assert np.array_equal(rep.output.astype(np.float32), ref_out)
    assert rep.overflow_events == row["overflow_events"]
    assert json.loads((FIX / "q.bin.meta.json").read_text())["distribution"] == "gaussian"
