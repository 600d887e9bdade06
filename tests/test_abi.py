"""The C-ABI library builds, loads without a GPU and exports every symbol include/fms.h declares;
the product package never imports the oracle (CPU only)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2007_14283_b200 import build
    build.build()
    import paper_2007_14283_b200 as fms
    return fms.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "fms.h")).read()
    return sorted(set(re.findall(r"\b(fms_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    so = os.path.join(ROOT, "paper_2007_14283_b200", "libfms.so")
    out = subprocess.check_output(["nm", "-D", "--defined-only", so], text=True)
    exported = set(re.findall(r" T (fms_\w+)", out))
    declared = _declared()
    assert declared and set(declared) <= exported, set(declared) - exported
    for name in declared:
        assert hasattr(lib, name)


def test_default_policy_matches_paper(lib):
    import paper_2007_14283_b200 as fms
    p = fms.default_policy()
    assert (p.kind, p.n_seeds, p.gamma, p.L, p.H, p.P) == (1, 128, 0.9, 2.0, 8.0, 0.99)


def test_no_device_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2007_14283_b200 as fms
    with pytest.raises(fms.FmsError):
        fms.Context(0)


def test_product_path_does_not_touch_oracle():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2007_14283_b200")):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "fms_oracle" not in txt and "fmso_" not in txt, fn


def test_sass_has_tcgen05_and_tma(lib):
    so = os.path.join(ROOT, "paper_2007_14283_b200", "libfms.so")
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", so], text=True)
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass and "STTM" in sass


def test_host_entry_rejects_bad_buffers_before_the_call():
    """Context.cluster_host checks dtype, device, contiguity and shapes before the
    raw pointers reach fms_cluster_batch_host (no GPU needed: the checks run first)."""
    import pytest
    import torch
    import paper_2007_14283_b200 as fms
    ctx = fms.Context.__new__(fms.Context)
    ctx.h = None
    e = torch.zeros((2, 10, 4), dtype=torch.float32)
    l = torch.zeros((2, 10), dtype=torch.int32)
    c = torch.zeros((2, 8, 4), dtype=torch.float32)
    with pytest.raises(TypeError):
        ctx.cluster_host(e.double(), l, c, 8)
    with pytest.raises(TypeError):
        ctx.cluster_host(e, l.long(), c, 8)
    with pytest.raises(TypeError):
        ctx.cluster_host(e.transpose(1, 2).contiguous().transpose(1, 2), l, c, 8)
    with pytest.raises(ValueError):
        ctx.cluster_host(e, torch.zeros((2, 9), dtype=torch.int32), c, 8)
    with pytest.raises(ValueError):
        ctx.cluster_host(e, l, c, 16)                      # centres_cap larger than the buffer
    with pytest.raises(ValueError):
        ctx.cluster_host(e, l, torch.zeros((2, 8, 3), dtype=torch.float32), 8)
    with pytest.raises(TypeError):
        ctx.cluster_host(e.numpy(), l, c, 8)
