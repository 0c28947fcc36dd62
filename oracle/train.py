"""Training of the P2S network -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's reference legs may use this module.

The paper trains "a small neural network to convert the coefficients from the Zernike
coefficients a_x ... to the PSF coefficients beta_x" (citing Mao et al. 2021)
without stating the loss or the optimiser.  Reading Q26: mean squared error over the
mini-batch and the K outputs,

    L = 1/(B K) sum_i sum_k (y_ik - beta_ik)^2,   y = W3 relu(W2 relu(W1 a + b1) + b2) + b3,

minimised by Adam (beta1 = 0.9, beta2 = 0.999, eps = 1e-8, bias-corrected moments), one
update per mini-batch; the sample order of every epoch is an input (`order`, epoch-major),
mini-batches are its consecutive chunks of `batch` samples (the last one may be shorter).
relu'(0) = 0.  Everything in fp64, written step by step: forward, the loss, backprop by the
chain rule, the Adam update.
"""
from __future__ import annotations

import numpy as np

ADAM_B1, ADAM_B2, ADAM_EPS = 0.9, 0.999, 1e-8


def forward(params, a):
    """params = [W1, b1, W2, b2, W3, b3]; a [B][n_in] -> (z1, h1, z2, h2, y)."""
    W1, b1, W2, b2, W3, b3 = params
    z1 = a @ W1.T + b1
    h1 = np.maximum(z1, 0.0)
    z2 = h1 @ W2.T + b2
    h2 = np.maximum(z2, 0.0)
    y = h2 @ W3.T + b3
    return z1, h1, z2, h2, y


def loss(params, a, beta) -> float:
    y = forward(params, a)[4]
    return float(np.mean((y - beta) ** 2))


def gradients(params, a, beta):
    """dL/dparams for the batch (a, beta), by the chain rule."""
    W1, b1, W2, b2, W3, b3 = params
    z1, h1, z2, h2, y = forward(params, a)
    B, K = beta.shape
    dy = 2.0 * (y - beta) / (B * K)
    dW3 = dy.T @ h2
    db3 = dy.sum(axis=0)
    dz2 = (dy @ W3) * (z2 > 0)
    dW2 = dz2.T @ h1
    db2 = dz2.sum(axis=0)
    dz1 = (dz2 @ W2) * (z1 > 0)
    dW1 = dz1.T @ a
    db1 = dz1.sum(axis=0)
    return [dW1, db1, dW2, db2, dW3, db3]


def adam_step(params, grads, m, v, t: int, lr: float):
    """One Adam update (t = 1, 2, ...), in place on params, m, v."""
    for p, g, mi, vi in zip(params, grads, m, v):
        mi *= ADAM_B1
        mi += (1.0 - ADAM_B1) * g
        vi *= ADAM_B2
        vi += (1.0 - ADAM_B2) * g * g
        mhat = mi / (1.0 - ADAM_B1 ** t)
        vhat = vi / (1.0 - ADAM_B2 ** t)
        p -= lr * mhat / (np.sqrt(vhat) + ADAM_EPS)


def train(layers, a, beta, order, epochs: int, batch: int, lr: float):
    """layers = [(W1, b1), (W2, b2), (W3, b3)]; a [n][n_in]; beta [n][K]; order [epochs][n].
    Returns (trained layers, per-epoch mean batch loss before each update, sample-weighted)."""
    params = [np.array(x, dtype=np.float64) for lw in layers for x in lw]
    a = np.asarray(a, np.float64)
    beta = np.asarray(beta, np.float64)
    order = np.asarray(order).reshape(epochs, -1)
    n = a.shape[0]
    m = [np.zeros_like(p) for p in params]
    v = [np.zeros_like(p) for p in params]
    t = 0
    curve = []
    for e in range(epochs):
        tot = 0.0
        for s in range(0, n, batch):
            idx = order[e, s:s + batch]
            ab, bb = a[idx], beta[idx]
            tot += loss(params, ab, bb) * len(idx)
            g = gradients(params, ab, bb)
            t += 1
            adam_step(params, g, m, v, t, lr)
        curve.append(tot / n)
    out = [(params[0], params[1]), (params[2], params[3]), (params[4], params[5])]
    return out, np.array(curve)
