"""Layer ComputeFeature / ComputeGradient definitions (oracle, float64).

Test infrastructure only.  PAPER.md §4.1.2: every layer has a
``ComputeFeature`` (forward) and a ``ComputeGradient`` (parameter gradients and
the source layer's gradient).  The paper names the layers (conv, pooling, LRN:
P:553; inner product / logistic: P:241; softmax cross-entropy loss: P:97, P:256;
Euclidean loss: P:326) but prints no formulas; the formulas are the textbook
definitions under the readings of SURVEY.md §8(c).3 (A4-A8), listed in
DESIGN.md.  Images are NHWC; conv weights [Cout][R][S][Cin]; IP weights
[d_v][d_h] (y = xW + b).

All functions take and return float64 numpy arrays.  No blocking, fusion or
reordering beyond the definitions: sums are written as loops over the filter
taps / windows with a numpy contraction over the remaining index.

Pins (tests/test_oracle_layers.py): pure-Python brute force on tiny shapes,
central finite differences, closed forms and SPEC examples
(S:129-141), torch-CPU-fp64 library routines (conv2d, max/avg_pool2d with
ceil_mode, local_response_norm) as independent cross-checks.
"""

import math

import numpy as np


# ----------------------------------------------------------------------------
# Convolution (reading A4: cross-correlation, zero padding, floor output size).
# ----------------------------------------------------------------------------
def conv_out_size(h, k, s, p):
    return (h + 2 * p - k) // s + 1


def conv_forward(x, W, b, stride, pad):
    """y[n,oh,ow,co] = b[co] + sum_{r,s,ci} W[co,r,s,ci] * x[n, oh*st-p+r, ow*st-p+s, ci]."""
    N, H, Wd, C = x.shape
    Co, R, S, C2 = W.shape
    assert C == C2
    Ho, Wo = conv_out_size(H, R, stride, pad), conv_out_size(Wd, S, stride, pad)
    xp = np.zeros((N, H + 2 * pad, Wd + 2 * pad, C))
    xp[:, pad:pad + H, pad:pad + Wd, :] = x
    y = np.zeros((N, Ho, Wo, Co))
    for r in range(R):
        for s in range(S):
            win = xp[:, r:r + stride * (Ho - 1) + 1:stride, s:s + stride * (Wo - 1) + 1:stride, :]
            y += np.tensordot(win, W[:, r, s, :], axes=([3], [1]))
    y += b[None, None, None, :]
    return y


def conv_backward(x, W, dy, stride, pad, need_dx=True):
    """dW[co,r,s,ci] = sum_{n,oh,ow} dy[n,oh,ow,co] x[n,oh*st-p+r,ow*st-p+s,ci];
    db[co] = sum dy; dx[n,h,w,ci] = sum over taps mapping onto (h,w) of dy*W."""
    N, H, Wd, C = x.shape
    Co, R, S, _ = W.shape
    Ho, Wo = dy.shape[1], dy.shape[2]
    xp = np.zeros((N, H + 2 * pad, Wd + 2 * pad, C))
    xp[:, pad:pad + H, pad:pad + Wd, :] = x
    dW = np.zeros_like(W)
    dxp = np.zeros_like(xp)
    for r in range(R):
        for s in range(S):
            sl = (slice(None), slice(r, r + stride * (Ho - 1) + 1, stride),
                  slice(s, s + stride * (Wo - 1) + 1, stride), slice(None))
            dW[:, r, s, :] = np.tensordot(dy, xp[sl], axes=([0, 1, 2], [0, 1, 2]))
            if need_dx:
                dxp[sl] += np.tensordot(dy, W[:, r, s, :], axes=([3], [0]))
    db = dy.sum(axis=(0, 1, 2))
    dx = dxp[:, pad:pad + H, pad:pad + Wd, :] if need_dx else None
    return dx, dW, db


# ----------------------------------------------------------------------------
# Pooling (reading A5: Caffe geometry, ceil mode, first-max tie-break).
# ----------------------------------------------------------------------------
def pool_out_size(h, k, s, p):
    ho = int(math.ceil((h + 2 * p - k) / s)) + 1
    if p > 0 and (ho - 1) * s >= h + p:
        ho -= 1
    return ho


def _window(o, k, s, p, h):
    start = o * s - p
    end = min(start + k, h + p)
    size = end - start
    return max(start, 0), min(end, h), size


def maxpool_forward(x, k, s, p):
    """y = max over the window; argmax = flat h*W+w of the FIRST maximum in
    row-major (h, then w) scan order with strict '>' from -inf (A5)."""
    N, H, W, C = x.shape
    Ho, Wo = pool_out_size(H, k, s, p), pool_out_size(W, k, s, p)
    y = np.full((N, Ho, Wo, C), -np.inf)
    idx = np.full((N, Ho, Wo, C), -1, dtype=np.int64)
    for oh in range(Ho):
        h0, h1, _ = _window(oh, k, s, p, H)
        for ow in range(Wo):
            w0, w1, _ = _window(ow, k, s, p, W)
            for h in range(h0, h1):
                for w in range(w0, w1):
                    v = x[:, h, w, :]
                    better = v > y[:, oh, ow, :]
                    y[:, oh, ow, :] = np.where(better, v, y[:, oh, ow, :])
                    idx[:, oh, ow, :] = np.where(better, h * W + w, idx[:, oh, ow, :])
    return y, idx


def maxpool_backward(x_shape, idx, dy):
    """dx[argmax] += dy (overlapping windows accumulate, ascending window order)."""
    N, H, W, C = x_shape
    dx = np.zeros((N, H * W, C))
    Ho, Wo = dy.shape[1], dy.shape[2]
    n_ix = np.arange(N)[:, None]
    c_ix = np.arange(C)[None, :]
    for oh in range(Ho):
        for ow in range(Wo):
            np.add.at(dx, (n_ix, idx[:, oh, ow, :], c_ix), dy[:, oh, ow, :])
    return dx.reshape(N, H, W, C)


def avgpool_forward(x, k, s, p):
    """y = (sum of in-bounds window) / pool_size, pool_size computed before
    clipping to the image (Caffe; equals the in-bounds count when p = 0)."""
    N, H, W, C = x.shape
    Ho, Wo = pool_out_size(H, k, s, p), pool_out_size(W, k, s, p)
    y = np.zeros((N, Ho, Wo, C))
    for oh in range(Ho):
        h0, h1, hs = _window(oh, k, s, p, H)
        for ow in range(Wo):
            w0, w1, ws = _window(ow, k, s, p, W)
            y[:, oh, ow, :] = x[:, h0:h1, w0:w1, :].sum(axis=(1, 2)) / (hs * ws)
    return y


def avgpool_backward(x_shape, dy, k, s, p):
    N, H, W, C = x_shape
    dx = np.zeros(x_shape)
    Ho, Wo = dy.shape[1], dy.shape[2]
    for oh in range(Ho):
        h0, h1, hs = _window(oh, k, s, p, H)
        for ow in range(Wo):
            w0, w1, ws = _window(ow, k, s, p, W)
            dx[:, h0:h1, w0:w1, :] += (dy[:, oh, ow, :] / (hs * ws))[:, None, None, :]
    return dx


# ----------------------------------------------------------------------------
# LRN across channels (reading A6).
# ----------------------------------------------------------------------------
def lrn_forward(x, n, alpha, beta, k):
    """scale_c = k + (alpha/n) sum_{|c'-c| <= n//2, 0<=c'<C} x_{c'}^2 ; y = x scale^-beta."""
    C = x.shape[-1]
    half = n // 2
    sq = x * x
    ssum = np.zeros_like(x)
    for c in range(C):
        lo, hi = max(0, c - half), min(C - 1, c + half)
        ssum[..., c] = sq[..., lo:hi + 1].sum(axis=-1)
    scale = k + (alpha / n) * ssum
    return x * scale ** (-beta), scale


def lrn_backward(x, y, scale, dy, n, alpha, beta):
    """dx_c = dy_c scale_c^-beta - (2 alpha beta / n) x_c sum_{|c'-c|<=n//2} dy_c' y_c' / scale_c'."""
    C = x.shape[-1]
    half = n // 2
    t = dy * y / scale
    tsum = np.zeros_like(x)
    for c in range(C):
        lo, hi = max(0, c - half), min(C - 1, c + half)
        tsum[..., c] = t[..., lo:hi + 1].sum(axis=-1)
    return dy * scale ** (-beta) - (2.0 * alpha * beta / n) * x * tsum


# ----------------------------------------------------------------------------
# Elementwise neurons.
# ----------------------------------------------------------------------------
def relu_forward(x):
    return np.maximum(x, 0.0)


def relu_backward(y, dy):
    """derivative 0 at 0 (reading A8): mask y > 0."""
    return dy * (y > 0)


def sigmoid_forward(x):
    """1/(1+e^-x), stable branch for x < 0."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def sigmoid_backward(y, dy):
    return dy * y * (1.0 - y)


# ----------------------------------------------------------------------------
# Inner product ("rotates (multiply W), shifts (plus b)").
# ----------------------------------------------------------------------------
def ip_forward(x, W, b):
    """y = x W + b, x [rows][d_v], W [d_v][d_h]."""
    return x @ W + b[None, :]


def ip_backward(x, W, dy, need_dx=True):
    """dW = x^T dy ; db = column sums of dy ; dx = dy W^T."""
    return (dy @ W.T if need_dx else None), x.T @ dy, dy.sum(axis=0)


# ----------------------------------------------------------------------------
# Loss layers (fused forward + backward).
# ----------------------------------------------------------------------------
def softmax_ce(z, labels, n_loc):
    """l_i = LSE(z_i) - z_{i,y_i}; dz = (softmax(z) - onehot(y)) / n_loc (S:149,
    readings A2, A7).  Returns (per-row losses, dz)."""
    C = z.shape[1]
    if np.any(labels < 0) or np.any(labels >= C):
        raise ValueError("label error: label outside [0, C)")
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    ssum = e.sum(axis=1, keepdims=True)
    lse = m[:, 0] + np.log(ssum[:, 0])
    rows = np.arange(z.shape[0])
    loss = lse - z[rows, labels]
    p = e / ssum
    dz = p.copy()
    dz[rows, labels] -= 1.0
    return loss, dz / n_loc


def euclidean(u, v, n_loc):
    """per-row 0.5*||u-v||^2 (L = (1/b) sum of these = (1/2b) sum ||u-v||^2);
    du = (u - v) / n_loc."""
    d = u - v
    return 0.5 * (d * d).sum(axis=1), d / n_loc
