"""CPU checks of the task-batched MAML network forms (maml.conv4_forward_tasks):
pure torch in float64, no CUDA library involved (the fused inner step is
replaced by the plain SGD-momentum recurrence)."""
import torch
import torch.nn.functional as F

from paper_2211_06934_b200 import maml

T = 3
SIZES = maml.sizes_of(maml.CONV4_SHAPES)


def _params(seed):
    g = torch.Generator().manual_seed(seed)
    phi = maml.init_params(0, "cpu").double()
    th = torch.stack([phi + 0.01 * torch.randn(phi.shape, generator=g, dtype=torch.float64)
                      for _ in range(T)])
    offs = [0]
    for n in SIZES:
        offs.append(offs[-1] + n)
    leaves = [th[:, a:b].reshape(T, *s) for a, b, s in zip(offs, offs[1:], maml.CONV4_SHAPES)]
    return th, leaves


def test_im2col_col2im_adjoint_pair_gradcheck():
    h = torch.randn(2, 3, 2, 5, 4, dtype=torch.float64, requires_grad=True)
    assert torch.autograd.gradcheck(maml._Im2Col.apply, (h,))
    assert torch.autograd.gradgradcheck(maml._Im2Col.apply, (h,))
    c = torch.randn(2, 27, 40, dtype=torch.float64, requires_grad=True)
    assert torch.autograd.gradcheck(lambda x: maml._Col2Im.apply(x, (2, 3, 2, 5, 4)), (c,))


def test_conv3x3_tasks_equals_conv2d():
    h = torch.randn(T, 4, 2, 7, 7, dtype=torch.float64)
    w = torch.randn(T, 5, 4, 3, 3, dtype=torch.float64)
    b = torch.randn(T, 5, dtype=torch.float64)
    out = maml._conv3x3_tasks(h, w, b)
    for t in range(T):
        ref = F.conv2d(h[t].transpose(0, 1), w[t], b[t], padding=1).transpose(0, 1)
        torch.testing.assert_close(out[t], ref, rtol=1e-12, atol=1e-12)


def test_task_batched_forms_equal_per_task_network():
    th, leaves = _params(1)
    data = [maml.task_data(0, t, "cpu") for t in range(T)]
    xs = torch.stack([d[0] for d in data], 1).flatten(1, 2).double()
    for net in ("cudnn", "gemm"):
        out = maml.conv4_forward_tasks(leaves, xs, T, net)
        for t in range(T):
            pt = [p.view(s) for p, s in zip(torch.split(th[t], SIZES), maml.CONV4_SHAPES)]
            ref = maml.conv4_forward(pt, data[t][0].double())
            torch.testing.assert_close(out[t], ref, rtol=1e-10, atol=1e-10)


def test_task_batched_second_order_meta_gradient_matches_per_task():
    """Sum over tasks of the 2-inner-step meta-gradients: task-batched gemm
    form == per-task loop (float64, plain SGD-momentum)."""
    cfg = maml.MamlConfig(tasks=T, inner_steps=2, net="gemm")
    phi = maml.init_params(0, "cpu").double()
    data = [[a.double() if a.is_floating_point() else a for a in maml.task_data(3, t, "cpu")]
            for t in range(T)]

    def torch_inner(g, b, theta):
        b1 = g if b is None else cfg.inner_momentum * b + g
        return theta - cfg.inner_lr * b1, b1

    mg, loss = maml.meta_grad_data(phi, data, cfg, torch_inner)

    class Inner:
        def __init__(self):
            self.T = T

        def __call__(self, g, b, theta):
            return torch_inner(g, b, theta)

    mg_b, loss_b = maml.meta_grad_batched(phi, data, cfg, Inner())
    torch.testing.assert_close(mg_b, mg, rtol=1e-9, atol=1e-12)
    torch.testing.assert_close(loss_b, loss, rtol=1e-12, atol=1e-12)
