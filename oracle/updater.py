"""Server-side Updater (oracle, float64).  Test infrastructure only.

PAPER.md §4.1.4: servers update Params with an updating protocol
(SGD, AdaGrad).  The plain SGD step is the commented Alg.:
Theta <- Theta - alpha * grad.  The north star adds gradient scale, momentum and
weight decay (reading A1, Caffe/SINGA form, lr inside the history):

    g' = s*g + lambda*lambda_scale*w
    v  = mu*v - eta_t*eta_scale*g'
    w  = w + v

with eta_t = eta_0 (fixed) or eta_0 * gamma^floor(t/T) (step).
At mu = 0 this is exactly SPEC S:406 value <- value - alpha*(grad + wd*value).

AdaGrad ("SINGA implements several parameter updating protocols, such as
AdaGrad"; reading A26 in DESIGN.md), with the same gradient
scale and weight decay as the SGD Updater:

    g' = s*g + lambda*lambda_scale*w
    h  = h + g'^2
    w  = w - eta_t*eta_scale * g' / (sqrt(h) + eps)

Pins (tests/test_oracle_updater_partition.py): S:409 (1.0, g 0.5, a 0.1 -> 0.95),
S:410 (g = 0 at wd = 0 -> unchanged), S:411 (alpha(250) = 0.25 alpha_0), the
constant-gradient momentum closed form, eta = 0 constancy, the lr / wd
multipliers against a rescaled base rate / decay; AdaGrad: S:418 (first step
-alpha*g/(|g| + eps)), S:419 (constant gradient 1: displacement
-alpha * sum_i 1/(sqrt(i) + eps)), S:420 (zero gradient: nothing changes).
"""

import numpy as np


def learning_rate(cfg, step):
    base = cfg["base_lr"]
    if cfg.get("lr_policy", "fixed") == "fixed":
        return base
    if cfg["lr_policy"] == "step":
        return base * cfg["gamma"] ** (step // cfg["step_size"])
    raise ValueError("unknown lr policy")


def sgd_momentum(w, v, g, cfg, step, grad_scale, lr_scale=1.0, wd_scale=1.0):
    """One update of (w, v) given the aggregated raw gradient g. Returns new (w, v)."""
    w = np.asarray(w, np.float64)
    v = np.asarray(v, np.float64)
    g = np.asarray(g, np.float64)
    eta = learning_rate(cfg, step) * lr_scale
    gp = grad_scale * g + cfg["weight_decay"] * wd_scale * w
    v_new = cfg["momentum"] * v - eta * gp
    return w + v_new, v_new


def adagrad(w, h, g, cfg, step, grad_scale, lr_scale=1.0, wd_scale=1.0):
    """One AdaGrad update of (w, h) given the aggregated raw gradient g."""
    w = np.asarray(w, np.float64)
    h = np.asarray(h, np.float64)
    g = np.asarray(g, np.float64)
    eta = learning_rate(cfg, step) * lr_scale
    gp = grad_scale * g + cfg["weight_decay"] * wd_scale * w
    h_new = h + gp * gp
    return w - eta * gp / (np.sqrt(h_new) + cfg.get("eps", 1e-8)), h_new


def update(w, state, g, cfg, step, grad_scale, lr_scale=1.0, wd_scale=1.0):
    """The configured Updater (cfg["type"]: "sgd_momentum" (default) or "adagrad")."""
    if cfg.get("type", "sgd_momentum") == "adagrad":
        return adagrad(w, state, g, cfg, step, grad_scale, lr_scale, wd_scale)
    return sgd_momentum(w, state, g, cfg, step, grad_scale, lr_scale, wd_scale)
