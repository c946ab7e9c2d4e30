"""GPU parity of the NEXT-4 entry points through the C ABI.

* jtfs_u2_map: the Fig. 1 scale-rate map |X * Psi| before Phi vs the
  oracle's u2_map, every psi_t path at c1 and sampled paths of a full-size c3 note;
  per-map relative L2 with the parity floor of tests/parity.py.
* jtfs_mulog_mu / jtfs_mulog_apply (Eqs. (adalog:mu), (adalog)) on seeded
  synthetic records (not GPU outputs), and jtfs_forward_mulog (mu-log fused into KE)
  vs the oracle's forward + mulog with a seeded mu; fused == unfused bit for bit.
"""
import numpy as np
import pytest

from oracle import jtfs_oracle as O
from paper_2204_08269_b200 import signals

from .parity import TOL, path_blocks, path_errors

pytestmark = pytest.mark.gpu

C1 = dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8)
C1E4 = dict(C1, average_fr=False)
C3 = dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)


@pytest.fixture(scope="module")
def jt():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a visible CUDA device")
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    return jtfs


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _map_errors(gpu_maps, ora_maps):
    norms = np.array([np.linalg.norm(m) for m in ora_maps])
    floor = 1e-3 * np.sqrt(np.mean(norms ** 2))
    return np.array([np.linalg.norm(g.astype(np.float64) - o) / max(np.linalg.norm(o), floor)
                     for g, o in zip(gpu_maps, ora_maps)])


@pytest.mark.parametrize("kw", [C1, C1E4], ids=["eq3", "eq4"])
def test_u2_map_c1_every_psi_t_path(jt, kw):
    up = signals.am_chirp(2 ** 10, 1024.0, 64.0, 8.0, 2.0)
    X = np.stack([up, signals.white(1, 2 ** 10, seed=9)[0]]).astype(np.float32)
    prm = O.Params(**kw)
    s = O.schedule(prm)
    plan = jt.Plan(**kw)
    x = _cuda(X)
    pis = [pi for pi, p in enumerate(s.paths) if p[0] in (O.SPIN, O.PSI_T_PHI_F)]
    for b in range(X.shape[0]):
        g = [plan.u2_map(x[b:b + 1], pi)[0].cpu().numpy() for pi in pis]
        o = [O.u2_map(X[b].astype(np.float64), prm, pi, s) for pi in pis]
        assert all(gi.shape == oi.shape for gi, oi in zip(g, o))
        e = _map_errors(g, o)
        assert e.max() <= TOL, (b, float(e.max()), pis[int(np.argmax(e))])
    # batched call == per-signal calls
    both = plan.u2_map(x, pis[0]).cpu().numpy()
    np.testing.assert_array_equal(both[1], plan.u2_map(x[1:2], pis[0])[0].cpu().numpy())


def test_u2_map_c3_full_size_sampled_paths(jt):
    # full-size note in the paper's c3 setting: the fastest alpha (largest map) and a slow one
    X = signals.notes(1)[0].astype(np.float32)
    prm = O.Params(**C3)
    s = O.schedule(prm)
    plan = jt.Plan(**C3)
    spin = [pi for pi, p in enumerate(s.paths) if p[0] == O.SPIN]
    pis = [spin[1], spin[-1], [pi for pi, p in enumerate(s.paths) if p[0] == O.PSI_T_PHI_F][0]]
    x = _cuda(X[None])
    g, o = [], []
    for pi in pis:
        g.append(plan.u2_map(x, pi)[0].cpu().numpy())
        o.append(O.u2_map(X.astype(np.float64), prm, pi, s))
    # floor from the sampled maps' RMS (maps of a note are within a few decades)
    e = _map_errors(g, o)
    assert e.max() <= TOL, e


def _synthetic_records(plan, B, seed):
    # seeded positive records in the out_3D layout (no GPU output feeds the oracle)
    L = plan.layout
    rng = np.random.default_rng(seed)
    S = rng.gamma(0.5, 1.0, size=(B, L.floats_per_signal)) * \
        np.exp(rng.uniform(-6, 2, size=(1, L.floats_per_signal)))
    return S.astype(np.float32)


def test_mulog_mu_and_apply_vs_oracle(jt):
    plan = jt.Plan(**C1)
    L = plan.layout
    B = 7
    S = _synthetic_records(plan, B, 3)
    S2 = S[:, L.off_s2:].reshape(B, L.n_paths, L.lambda_out, L.n_frames).astype(np.float64)
    mu_ref = O.mulog_mu(S2)
    mu = plan.mulog_mu(_cuda(S)).cpu().numpy()
    np.testing.assert_allclose(mu, mu_ref, rtol=2e-7)
    # deterministic
    assert np.array_equal(mu, plan.mulog_mu(_cuda(S)).cpu().numpy())
    mu32 = mu_ref.astype(np.float32)
    mu32[3] = 0.0                                        # a silent path maps to 0
    out = plan.mulog_apply(_cuda(S), _cuda(mu32), 0.1).cpu().numpy()
    ref = O.mulog(S2, mu32.astype(np.float64), 0.1)
    np.testing.assert_array_equal(out[:, :L.off_s2], S[:, :L.off_s2])      # S0/S1 untouched (R22)
    got = out[:, L.off_s2:].reshape(ref.shape)
    assert np.all(got[:, 3] == 0)
    np.testing.assert_allclose(got, ref, rtol=3e-6, atol=1e-30)
    # in place
    Sx = _cuda(S)
    plan.mulog_apply(Sx, _cuda(mu32), 0.1, out=Sx)
    np.testing.assert_array_equal(Sx.cpu().numpy(), out)


@pytest.mark.parametrize("kw", [C1, C1E4], ids=["eq3", "eq4"])
def test_forward_mulog_vs_oracle_and_unfused(jt, kw):
    import torch
    up = signals.am_chirp(2 ** 10, 1024.0, 64.0, 8.0, 2.0)
    X = np.stack([up, up[::-1].copy(), signals.white(1, 2 ** 10, seed=5)[0]]).astype(np.float32)
    prm = O.Params(**kw)
    s = O.schedule(prm)
    plan = jt.Plan(**kw)
    rng = np.random.default_rng(11)
    mu = np.exp(rng.uniform(-3, 1, size=len(s.paths))).astype(np.float32)   # seeded mu
    x, mud = _cuda(X), _cuda(mu)
    fused = plan.forward_mulog(x, mud, 0.1)
    unfused = plan.mulog_apply(plan.forward(x), mud, 0.1)
    torch.cuda.synchronize()
    assert torch.equal(fused, unfused)                   # bit-identical
    for b in range(X.shape[0]):
        ref = O.jtfs_forward(X[b].astype(np.float64), prm, s=s)
        S2t = O.mulog(ref["S2"][None], mu.astype(np.float64), 0.1)[0]
        s0, s1, s2 = plan.unpack(fused[b].cpu().numpy().astype(np.float64))
        e = path_errors(path_blocks(s0, s1, s2), path_blocks(ref["S0"], ref["S1"], S2t))
        assert e.max() <= TOL, (b, float(e.max()), int(np.argmax(e)))
