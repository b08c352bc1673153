"""GP hyperparameter learning (Alg.1 "Learn GP transition dynamics using D"; Eq.5-6,
P:77-80): maximise the exact log marginal likelihood of each output GP
by Adam on the log-hyperparameters phi = [log l (d) | log s | log sn2] (lr 0.05, at
most 500 steps, stop when the gradient's inf-norm < 1e-4 or the likelihood stops improving).

Both the objective/gradient (``gp_log_marginal_likelihood``: fp64 Cholesky, triangular inverse
and the fused Khat^-1 x dKhat reduction; or, at large N, ``gp_log_marginal_likelihood_bbmm``: the
stochastic BBMM estimate GPyTorch uses, readings R39 / R40) and the Adam update
(``policy_adam_step``) run in libbagel.so; this module only marshals the d + 2 numbers per step.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass
class FitLog:
    mll: list = field(default_factory=list)
    grad_inf: list = field(default_factory=list)
    steps: int = 0


def fit_hyperparameters(ctx, m: int, log_hyp0=None, iters: int = 500, lr: float = 0.05,
                        tol_grad: float = 1e-4, tol_rel: float = 1e-9, window: int = 10, bbmm=None):
    """Maximise log p(y_m | X, phi) for output m of the loaded GP.  Returns (phi [float64 numpy],
    FitLog).  log_hyp0 None starts from the loaded hyperparameters.  bbmm None uses the exact
    objective; a dict (n_probes, n_iter, precond_rank, seed) uses the BBMM estimate instead, with a
    fresh probe stream (seed + step) every step, as stochastic-gradient training does -- the
    stopping rules then see a noisy objective, so give a fixed iteration budget.  Apply the result with
    ``ctx.gp_load(X, Y, exp(phi[:d]), exp(phi[d]), exp(phi[d + 1]))`` (per output) and rebuild the
    LOVE cache."""
    phi = torch.as_tensor(np.asarray(log_hyp0 if log_hyp0 is not None else ctx.loaded_log_hyp(m),
                                     dtype=np.float32), device=ctx.dev).clone()
    m1, m2 = torch.zeros_like(phi), torch.zeros_like(phi)
    g_dev = torch.empty_like(phi)
    log = FitLog()
    for t in range(1, int(iters) + 1):
        h = phi.cpu().numpy().astype(np.float64)
        if bbmm is None:
            val, g = ctx.log_marginal_likelihood(m, h, want_grad=True)
        else:
            val, g, _ = ctx.log_marginal_likelihood_bbmm(
                m, h, n_probes=bbmm.get("n_probes", 8), n_iter=bbmm.get("n_iter", 100),
                seed=bbmm.get("seed", 0) + t, precond_rank=bbmm.get("precond_rank", 16))
        log.mll.append(val)
        log.grad_inf.append(float(np.abs(g).max()))
        if log.grad_inf[-1] < tol_grad:
            break
        if len(log.mll) > window and abs(log.mll[-1] - log.mll[-1 - window]) <= tol_rel * abs(log.mll[-1]):
            break
        g_dev.copy_(torch.from_numpy((-g).astype(np.float32)))  # Adam minimises -log p
        ctx.adam_step(phi, g_dev, m1, m2, t, lr)
        log.steps = t
    return phi.cpu().numpy().astype(np.float64), log
