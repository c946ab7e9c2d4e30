"""Texture resynthesis by gradient descent through the JTFS.

E(y) = ||S x - S y|| / ||S x||; the gradient comes from the C ABI's jtfs_backward
(every stage the exact adjoint of the forward kernels); the step size follows the
bold driver heuristic (grow on success, shrink and retry on failure).
The paper's update reads y + mu grad E; descent needs the minus sign.
Plumbing only: all arithmetic of S and its adjoint runs in libjtfs.so.
"""
from __future__ import annotations


def loss_and_grad(plan, Sx, y):
    """E(y) and dE/dy for y (CUDA float32 [1, N]), Sx the target record [1, F]: forward,
    the fused loss kernel (jtfs_resynth_loss: E and dE/dSy) and jtfs_backward, all in
    libjtfs.so; E is read back for the bold driver's accept / reject decision."""
    Sy = plan.forward(y)
    E, dout = plan.resynth_loss(Sy, Sx)
    return float(E.item()), plan.backward(y, dout)


def resynthesize(plan, x, y0, iters: int, mu0: float | None = None, up: float = 1.2, down: float = 0.5):
    """Bold-driver gradient descent from y0 towards the JTFS of x.  Returns (y, [E_n])."""
    import torch
    Sx = plan.forward(x).clone()
    y = y0.clone().contiguous()
    E, g = loss_and_grad(plan, Sx, y)
    # initial step: move y by ~10 % of its norm
    mu = mu0 if mu0 is not None else float(0.1 * y.norm() / max(g.norm().item(), 1e-30))
    hist = [E]
    for _ in range(iters):
        cand = (y - mu * g).contiguous()
        Ec, gc = loss_and_grad(plan, Sx, cand)
        if Ec < E:
            y, E, g, mu = cand, Ec, gc, mu * up
        else:
            mu *= down
        hist.append(E)
    torch.cuda.synchronize()
    return y, hist
