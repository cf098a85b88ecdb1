"""CPU-side checks of the C-ABI boundary: the library loads without a GPU and
exports every function include/dsg.h declares; calls fail loudly (no
fallback) when no device is present."""
import ctypes
import os
import re

import pytest

from paper_2509_12138_b200 import api
from paper_2509_12138_b200.types import DsplatError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dsg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("dsg_render", "dsg_backward", "dsg_masked_loss", "dsg_adam_step", "dsg_train",
              "dsg_render_mask", "dsg_views_synthesize", "dsg_knn_mean", "dsg_seed_gaussians"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = api.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version():
    assert api.lib().dsg_abi_version() == 1


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    with pytest.raises(DsplatError, match="InvalidArgument"):
        api.Context(0)
