"""Host-side checks of the functional layer (no GPU): input validation runs
before any pointer reaches the C ABI, and update()'s flat-buffer rule."""
import pytest
import torch

import paper_2211_06934_b200 as pkg
from paper_2211_06934_b200 import functional as F


def _cfg(n):
    return F.StepConfig(pkg.Tree(numel=n))


def test_cpu_gradient_rejected_before_the_c_call():
    g = torch.zeros(16)
    with pytest.raises(TypeError, match="CUDA"):
        pkg.AdamStep.apply(g, None, None, None, 1e-3, 0.9, 0.999, 1e-8, 1, 0.0, _cfg(16))
    with pytest.raises(TypeError, match="CUDA"):
        pkg.functional.SgdStep.apply(g, None, None, 1e-3, 0.0, False, _cfg(16))


def test_validation_messages(monkeypatch):
    cfg = _cfg(16)
    # exercise the dtype / size / device rules through the checker directly
    g = torch.zeros(16)
    monkeypatch.setattr(torch.Tensor, "is_cuda", property(lambda self: True))
    F._check_args(cfg, g, (None, torch.zeros(16, dtype=torch.bfloat16)), (torch.zeros(16),))
    with pytest.raises(TypeError, match="float32"):
        F._check_args(cfg, g.double())
    with pytest.raises(ValueError, match="elements"):
        F._check_args(cfg, torch.zeros(15))
    with pytest.raises(TypeError, match="dtype"):
        F._check_args(cfg, g, (torch.zeros(16, dtype=torch.float16),))
    with pytest.raises(ValueError, match="elements"):
        F._check_args(cfg, g, (), (torch.zeros(17),))
    with pytest.raises(TypeError, match="dtype"):
        F._check_args(cfg, g, (), (torch.zeros(16, dtype=torch.bfloat16),))
    with pytest.raises(ValueError, match="per leaf"):
        F._check_args(cfg, g, lr_leaf=torch.zeros(2))
    with pytest.raises(TypeError, match="lr_leaf"):
        F._check_args(cfg, g, lr_leaf=torch.zeros(1, dtype=torch.float64))


def test_flat_buffer_rule():
    layout = F.FlatTree([(3, 4), (5,)], device="cpu")
    assert F._is_flat(torch.zeros(17), layout)
    assert not F._is_flat([torch.zeros(3, 4), torch.zeros(5)], layout)
    with pytest.raises(ValueError, match="flat buffer"):
        F._is_flat(torch.zeros(3, 4), layout)
    one = F.FlatTree([(3, 4)], device="cpu")
    assert F._is_flat(torch.zeros(3, 4), one)
    assert F._is_flat(torch.zeros(12), one)
