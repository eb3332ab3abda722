"""Pins of the oracle's NEXT-3 training pieces (Eq. 2 P:131,
"optimized via stochastic gradient descent on image reconstruction losses"): the L1 loss
gradient and the Adam step on raw (log-scale / logit-opacity / identity) parameters.

Pinned against library routines (torch CPU autograd and torch.optim.Adam, float64) and the
closed form of Adam's first step (|update| = lr when eps = 0)."""
import numpy as np
import torch

import oracle


def test_l1_matches_torch_autograd():
    rng = np.random.default_rng(0)
    img = rng.uniform(0, 1, (3, 17, 23)).astype(np.float32)
    gt = rng.uniform(0, 1, (3, 17, 23)).astype(np.float32)
    gt[0, :3] = img[0, :3]                        # exact ties: gradient 0
    L, g = oracle.l1_loss_grad(img, gt)
    ti = torch.tensor(img, dtype=torch.float64, requires_grad=True)
    tl = torch.nn.functional.l1_loss(ti, torch.tensor(gt, dtype=torch.float64))
    tl.backward()
    assert abs(L - tl.item()) <= 1e-12
    assert np.array_equal(g, ti.grad.numpy().astype(np.float32))
    assert np.all(g[0, :3] == 0)


def test_adam_first_step_closed_form():
    """t = 1, eps = 0: m_hat = g, v_hat = g^2, so raw moves by exactly -lr sign(g)."""
    g = np.array([0.3, -2.0, 1e-6, -1e-3])
    raw = np.array([1.0, 2.0, 3.0, 4.0])
    m, v = np.zeros(4), np.zeros(4)
    oracle.adam_step(g, raw, m, v, 0, 0.01, eps=0.0, t=1)
    assert np.allclose(raw, [0.99, 2.01, 2.99, 4.01], rtol=0, atol=1e-15)


def test_adam_matches_torch_optim_with_activations():
    """Five steps on three groups (identity, exp, sigmoid), per-group learning rates:
    the oracle's raw parameters / activations equal torch.optim.Adam on the raw tensor with
    the chain-rule gradient from torch autograd of the activation."""
    rng = np.random.default_rng(1)
    n = 50
    groups = [(0, 1.6e-4, lambda p: p), (1, 5e-3, torch.exp), (2, 5e-2, torch.sigmoid)]
    for act, lr, fn in groups:
        raw0 = rng.normal(0, 1, n)
        raw = raw0.copy()
        m, v = np.zeros(n), np.zeros(n)
        p = torch.tensor(raw0, dtype=torch.float64, requires_grad=True)
        opt = torch.optim.Adam([p], lr=lr, betas=(0.9, 0.999), eps=1e-15)
        for t in range(1, 6):
            g_act = rng.normal(0, 1, n)
            out = oracle.adam_step(g_act, raw, m, v, act, lr, t=t)
            opt.zero_grad()
            fn(p).backward(torch.tensor(g_act, dtype=torch.float64))
            opt.step()
            assert np.allclose(raw, p.detach().numpy(), rtol=1e-12, atol=1e-14), (act, t)
            assert np.allclose(out, fn(p.detach()).numpy(), rtol=1e-12, atol=1e-14)
