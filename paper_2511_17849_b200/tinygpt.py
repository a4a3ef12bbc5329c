"""GPU forward/backward of the reference's desk model -- the
gradient source for closed-loop runs without CPU gradients.

A torch restatement of model.py:79-384: byte-level pre-norm transformer,
learned positions, causal multi-head attention, 2x MLP with tanh-GELU, tied
output head, LayerNorm eps 1e-5, mean next-token cross-entropy.  Parameters are
views into one flat vector in the reference layout (model.py:79-94), so the
optimizer engine works on the same flat buffer the reference's optimizer sees.
Backward is autograd (the reference's manual backward computes the same
gradient; in fp64 the two agree to 1e-16, in fp32 to rounding).  This is the
model, not the optimizer hot path: plain torch ops, no custom kernels.
"""

from __future__ import annotations

import math

import numpy as np
import torch

LN_EPS = 1e-5
GELU_C = math.sqrt(2.0 / math.pi)
GELU_A = 0.044715


def param_shapes(vocab: int, d: int, layers: int, seq: int):
    """model.py:79-94."""
    f = 2 * d
    shapes = [("wte", (vocab, d)), ("wpe", (seq, d))]
    for i in range(layers):
        p = f"h{i}."
        shapes += [(p + "ln1_g", (d,)), (p + "ln1_b", (d,)), (p + "w_qkv", (d, 3 * d)), (p + "b_qkv", (3 * d,)),
                   (p + "w_attn_out", (d, d)), (p + "b_attn_out", (d,)), (p + "ln2_g", (d,)), (p + "ln2_b", (d,)),
                   (p + "w_fc", (d, f)), (p + "b_fc", (f,)), (p + "w_proj", (f, d)), (p + "b_proj", (d,))]
    shapes += [("lnf_g", (d,)), ("lnf_b", (d,))]
    return shapes


def unflatten(theta: torch.Tensor, shapes):
    out, off = {}, 0
    for name, shp in shapes:
        n = math.prod(shp)
        out[name] = theta[off: off + n].view(shp)
        off += n
    return out


def _ln(x, g, b):
    mu = x.mean(-1, keepdim=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdim=True)
    return xc / torch.sqrt(var + LN_EPS) * g + b


def _gelu(u):
    # model.py:198-218: 0.5*u*(1+tanh(c*(u + a*u^3)))
    return 0.5 * u * (1.0 + torch.tanh(GELU_C * (u + GELU_A * u * u * u)))


def loss_fn(theta: torch.Tensor, batch: torch.Tensor, cfg: dict) -> torch.Tensor:
    """Mean CE of batch[:, 1:] given batch[:, :-1] (model.py:241-306)."""
    d, H, L_ = cfg["d"], cfg["heads"], cfg["layers"]
    shapes = param_shapes(cfg["vocab"], d, L_, cfg["seq"])
    p = unflatten(theta, shapes)
    tok_in, tok_out = batch[:, :-1], batch[:, 1:]
    B, T = tok_in.shape
    hd = d // H
    x = p["wte"][tok_in] + p["wpe"][:T]
    mask = torch.full((T, T), float("-inf"), device=theta.device).triu(1)
    for i in range(L_):
        q_ = f"h{i}."
        n1 = _ln(x, p[q_ + "ln1_g"], p[q_ + "ln1_b"])
        qkv = n1.reshape(-1, d) @ p[q_ + "w_qkv"] + p[q_ + "b_qkv"]
        qkv = qkv.reshape(B, T, 3, H, hd).permute(2, 0, 3, 1, 4)
        q, k, v = qkv[0], qkv[1], qkv[2]
        att = (q @ k.transpose(-1, -2)) * (1.0 / math.sqrt(hd)) + mask
        att = torch.softmax(att, dim=-1)
        ctx = (att @ v).permute(0, 2, 1, 3).reshape(B, T, d)
        x = x + (ctx.reshape(-1, d) @ p[q_ + "w_attn_out"] + p[q_ + "b_attn_out"]).reshape(B, T, d)
        n2 = _ln(x, p[q_ + "ln2_g"], p[q_ + "ln2_b"])
        h = _gelu(n2.reshape(-1, d) @ p[q_ + "w_fc"] + p[q_ + "b_fc"])
        x = x + (h @ p[q_ + "w_proj"] + p[q_ + "b_proj"]).reshape(B, T, d)
    nf = _ln(x, p["lnf_g"], p["lnf_b"])
    logits = nf.reshape(-1, d) @ p["wte"].T
    return torch.nn.functional.cross_entropy(logits, tok_out.reshape(-1))


def loss_and_grad(theta: torch.Tensor, batch: torch.Tensor, cfg: dict, grad_out: torch.Tensor):
    """Loss (python float) and gradient written into ``grad_out`` (flat fp32)."""
    th = theta.detach().requires_grad_(True)
    loss = loss_fn(th, batch, cfg)
    (g,) = torch.autograd.grad(loss, th)
    grad_out.copy_(g)
    return float(loss.item())


def init_params(vocab: int, d: int, layers: int, seq: int, seed_or_rng, dtype=np.float32) -> np.ndarray:
    """model.py:122-141 with the same RNG stream: weights and embeddings
    N(0, 0.02^2) drawn in layout order, LayerNorm gains 1, biases 0.  The
    reference seeds it with ``default_rng([seed, 100])`` (driver.py:264)."""
    rng = seed_or_rng if isinstance(seed_or_rng, np.random.Generator) else np.random.default_rng(seed_or_rng)
    dt = np.dtype(dtype)
    shapes = param_shapes(vocab, d, layers, seq)
    theta = np.zeros(sum(math.prod(s) for _, s in shapes), dtype=dt)
    off = 0
    for name, shp in shapes:
        n = math.prod(shp)
        base = name.rsplit(".", 1)[-1]
        view = theta[off: off + n].reshape(shp)
        if base.startswith("w") or name in ("wte", "wpe"):
            view[...] = rng.standard_normal(shp, dtype=dt) * dt.type(0.02)
        elif base.endswith("_g"):
            view[...] = 1.0
        off += n
    return theta
