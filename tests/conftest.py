"""Shared pytest wiring: markers, repo on sys.path, golden fixture loader."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_cases() -> list[str]:
    return sorted(p.stem for p in GOLDEN.glob("attn_*.npz"))


BASELINE_REF = ROOT / "baseline" / "_ref"


def lpattn_path():
    """Where the unmodified reference package can be imported from: the pip-installed copy in
    baseline/_ref (travels to the GPU box) or the read-only source tree (build container)."""
    for p in (BASELINE_REF, REF_SRC):
        if (p / "lpattn" / "__init__.py").exists():
            return p
    return None


def reference_available() -> bool:
    return (REF_SRC / "lpattn" / "__init__.py").exists()


@pytest.fixture(scope="session")
def lpattn():
    """The unmodified reference package, only where it exists (build container)."""
    if not reference_available():
        pytest.skip("reference source tree not present on this machine")
    sys.path.insert(0, str(REF_SRC))
    import lpattn as mod
    return mod


def golden_config(g):
    """(seq, dim, heads, causal, smoothing, qk_bits, pv, depth, waive, p_r, v_r, sm_scale) of a fixture."""
    seq, dim, heads, causal, smoothing, qk_bits, fp16, depth, waive = (int(x) for x in g["cfg"])
    p_r, v_r, sm = (float(x) for x in g["ranges"])
    return dict(seq=seq, dim=dim, heads=heads, causal=bool(causal), smoothing=bool(smoothing),
                qk_bits=qk_bits, pv="fp16" if fp16 else "fp32", depth=depth, waive=bool(waive),
                p_r=p_r, v_r=v_r, sm_scale=None if sm < 0 else sm)


def gpu_ready() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
