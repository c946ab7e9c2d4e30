"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Intermediate taps (X_hat, U1, Y2, Y_phi) and the full out_3D record, on seeded
synthetic inputs shaped like the paper's workloads: AM/FM chirps
(Eq. (5)), notes, white noise; Eq. (3) and Eq. (4); reflect and periodic
padding; ragged batches; determinism.  Bar: per-path relative L2 <= 1e-4
(tests/parity.py).
"""
import numpy as np
import pytest

from oracle import jtfs_oracle as O
from paper_2204_08269_b200 import signals

from .parity import TOL, path_blocks, path_errors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def jt():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a visible CUDA device")
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    return jtfs


def _run(jt, kw, X):
    import torch
    plan = jt.Plan(**kw)
    x = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).cuda()
    out = plan.forward(x)
    torch.cuda.synchronize()
    return plan, out


def _check_signal(plan, out_row, x64, prm, paths=None, tol=TOL):
    s = O.schedule(prm)
    ref = O.jtfs_forward(x64, prm, paths=paths, s=s)
    s0, s1, s2 = plan.unpack(out_row.cpu().numpy().astype(np.float64))
    g = path_blocks(s0, s1, s2)
    o = path_blocks(ref["S0"], ref["S1"], ref["S2"])
    n_first = 1 + s.n1
    sel = list(range(n_first)) + [n_first + p for p in (paths if paths is not None else range(len(s.paths)))]
    e = path_errors(g, o, sel)
    assert e.max() <= tol, (float(e.max()), int(np.argmax(e)), sel[int(np.argmax(e))])
    return e


C1 = dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8)


def _c1_inputs():
    up = signals.am_chirp(2 ** 10, 1024.0, 64.0, 8.0, 2.0)
    return np.stack([up, up[::-1].copy(), signals.white(1, 2 ** 10, seed=5)[0],
                     signals.am_chirp(2 ** 10, 1024.0, 200.0, 30.0, -1.0)])


def test_tap_xhat_and_scalogram(jt):
    import torch
    prm = O.Params(**C1)
    s = O.schedule(prm)
    X = _c1_inputs()
    plan = jt.Plan(**C1)
    x = torch.from_numpy(X).cuda()
    xh = plan.debug_tap(0, x).cpu().numpy().view(np.complex64).reshape(len(X), s.N_pad)
    u1 = plan.debug_tap(1, x).cpu().numpy().reshape(len(X), -1)
    y2 = plan.debug_tap(2, x).cpu().numpy().reshape(len(X), -1)
    yp = plan.debug_tap(3, x).cpu().numpy().reshape(len(X), s.n1, -1)
    for b in range(len(X)):
        x64 = X[b].astype(np.float64)
        ref = np.fft.fft(O.pad_signal(x64, s))
        assert np.abs(xh[b] - ref).max() <= 1e-5 * np.abs(ref).max()
        S0, S1, Yphi, U1hat, Y2 = O.first_order(x64, s)
        # scalogram rows U1_lambda: per-row relative L2 with the parity floor (tests/parity.py)
        rows_o = [np.fft.ifft(U1hat[lam]).real for lam in range(s.n1)]
        offs = np.cumsum([0] + [len(r) for r in rows_o])
        rows_g = [u1[b, offs[i]:offs[i + 1]] for i in range(s.n1)]
        e = path_errors(rows_g, rows_o)
        assert e.max() <= 1e-5, (float(e.max()), int(np.argmax(e)))
        # Y2 rows (lambda, alpha)
        rows_o, rows_g, off = [], [], 0
        for a in s.alphas:
            ref2 = Y2[a]
            pl = y2[b, off:off + 2 * ref2.size].reshape(2 * ref2.shape[0], ref2.shape[1])
            g2 = pl[0::2] + 1j * pl[1::2]            # planar rows: re, im
            rows_o += list(ref2)
            rows_g += list(g2)
            off += 2 * ref2.size
        e = path_errors(rows_g, rows_o)
        assert e.max() <= 1e-5, (float(e.max()), int(np.argmax(e)))
        assert np.abs(yp[b] - Yphi).max() <= 1e-5 * np.abs(Yphi).max()


@pytest.mark.parametrize("variant", ["eq3", "eq4", "periodic", "periodic_eq4"])
def test_c1_full_parity(jt, variant):
    kw = dict(C1)
    if "eq4" in variant:
        kw["average_fr"] = False
    if "periodic" in variant:
        kw["pad_mode"] = jt.JTFS_PAD_PERIODIC
    prm = O.Params(**{k: v for k, v in kw.items() if k != "pad_mode"},
                   pad="periodic" if "periodic" in variant else "reflect")
    X = _c1_inputs()
    plan, out = _run(jt, kw, X)
    for b in range(len(X)):
        _check_signal(plan, out[b], X[b].astype(np.float64), prm)


def test_c1_spin_selectivity_on_gpu(jt):
    # Fig. 1: theta=-1 energy dominates for the up-chirp, theta=+1 for the reversal
    X = _c1_inputs()[:2]
    plan, out = _run(jt, C1, X)
    _, _, s2 = plan.unpack(out.cpu().numpy().astype(np.float64))
    paths = plan.paths()
    e = np.zeros((2, 2))
    for i, (k, th, *_r) in enumerate(paths):
        if k == jt.PATH_SPIN:
            e[:, (th + 1) // 2] += (s2[:, i] ** 2).sum(axis=(1, 2))
    assert e[0, 0] / e[0, 1] > 2.0 and e[1, 0] / e[1, 1] < 0.5


def test_c2_chirp_grid_parity(jt):
    kw = dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False)
    prm = O.Params(**kw)
    _, sig = signals.chirp_grid(n=4)   # corners + interior of the 16^3 ranges
    X = sig[[0, 21, 42, 63]]
    plan, out = _run(jt, kw, X)
    for b in range(len(X)):
        _check_signal(plan, out[b], X[b].astype(np.float64), prm)


def test_c3_full_size_sampled_paths(jt):
    # BASELINE config c3 (N=2^16, J=12, Q=16, J_fr=5, T=2^13, F=4) in bench's launch
    # configuration; oracle on a sample of paths of two notes.
    kw = dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
    prm = O.Params(**kw)
    X = signals.notes(3, seed0=1000)
    plan, out = _run(jt, kw, X)
    s = O.schedule(prm)
    P = len(s.paths)
    sample = sorted({0, 5, 59, 60, 61, 119, P - 17, P - 8, P - 7, P - 2, P - 1})
    for b in (0, 2):
        O.set_workers(8)
        _check_signal(plan, out[b], X[b].astype(np.float64), prm, paths=sample)


@pytest.mark.parametrize("kw", [C1, dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False),
                                dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)], ids=["c1", "c2", "c3"])
def test_kd_tensor_core_matches_simt(jt, kw):
    # consistency (not parity) check: the tcgen05 fp16-split contraction against the FP32
    # SIMT validation kernel (plan flag JTFS_KD_SIMT) on the same inputs
    import torch
    X = signals.notes(2, N=kw["N"], seed0=77) if kw["N"] >= 2 ** 13 else _c1_inputs()
    x = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    a = jt.Plan(**kw, flags=jt.JTFS_KD_SIMT).forward(x).cpu().numpy().astype(np.float64)
    b = jt.Plan(**kw).forward(x).cpu().numpy().astype(np.float64)
    for i in range(len(X)):
        assert np.linalg.norm(a[i] - b[i]) <= 1e-5 * np.linalg.norm(a[i])


@pytest.mark.parametrize("kw", [dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False),
                                dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)], ids=["c2", "c3"])
def test_kd_cta_pairs_match_single_ctas(jt, kw):
    # the cta_group::2 KD (CTA pairs, M = 256) against the single-CTA KD (plan flag
    # JTFS_KD_NOPAIR): same fp16 operands and per-row K order, so equal up to the order of
    # the epilogue's fp32 sums (in practice bit-identical)
    import torch
    X = signals.notes(5, N=kw["N"], seed0=313)
    x = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    a = jt.Plan(**kw, flags=jt.JTFS_KD_NOPAIR).forward(x).cpu().numpy().astype(np.float64)
    b = jt.Plan(**kw).forward(x).cpu().numpy().astype(np.float64)
    for i in range(len(X)):
        assert np.linalg.norm(a[i] - b[i]) <= 1e-6 * np.linalg.norm(a[i])


def test_determinism_and_batch_independence(jt):
    import torch
    X = np.concatenate([_c1_inputs(), signals.white(37, 2 ** 10, seed=9)])
    plan = jt.Plan(**C1)
    x = torch.from_numpy(X).cuda()
    a = plan.forward(x).cpu().numpy()
    b = plan.forward(x).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    c = plan.forward(x[3:4].contiguous()).cpu().numpy()
    assert np.array_equal(a[3:4].view(np.uint32), c.view(np.uint32))


def test_edge_cases(jt):
    import torch
    plan = jt.Plan(**C1)
    x = torch.zeros(0, C1["N"], device="cuda")
    assert plan.forward(x).shape == (0, plan.floats_per_signal)
    z = plan.forward(torch.zeros(2, C1["N"], device="cuda"))
    assert torch.count_nonzero(z).item() == 0                   # zero -> zero
    pf = jt.Plan(**C1, flags=jt.JTFS_CHECK_FINITE)
    xb = torch.zeros(1, C1["N"], device="cuda")
    xb[0, 7] = float("nan")
    with pytest.raises(jt.JTFSError) as e:
        pf.forward(xb)
    assert e.value.status == jt.JTFS_ERR_NONFINITE
    lib = jt.library()
    out = torch.empty(1, plan.floats_per_signal, device="cuda")
    ws = torch.empty(plan.workspace_size(1), dtype=torch.uint8, device="cuda")
    st = lib.jtfs_forward(plan.handle, xb.data_ptr(), 1, out.data_ptr(), ws.data_ptr(), 64, None)
    assert st == jt.JTFS_ERR_WORKSPACE


P42 = dict(N=2 ** 16, J=13, Q=16, J_fr=6, T=2 ** 11, F=4)   # Sec. 4.2 preset: 44 x 32 per path


def test_paper_preset_sampled_paths(jt):
    # the paper's convnet setting (32 frames: the NF = 32 tensor-core KD variant); oracle on a
    # sample of paths of one note, the S0 / S1 rows in full
    prm = O.Params(**P42)
    X = signals.notes(2, seed0=2000)
    plan, out = _run(jt, P42, X)
    s = O.schedule(prm)
    assert (s.lam_out, s.n_frames) == (44, 32)
    P = len(s.paths)
    sample = sorted({0, 7, 63, 64, P // 2, P - 20, P - 9, P - 8, P - 2, P - 1})
    O.set_workers(8)
    _check_signal(plan, out[1], X[1].astype(np.float64), prm, paths=sample)


def test_kd_tensor_core_matches_simt_paper_preset(jt):
    import torch
    X = signals.notes(2, seed0=91)
    x = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    a = jt.Plan(**P42, flags=jt.JTFS_KD_SIMT).forward(x).cpu().numpy().astype(np.float64)
    b = jt.Plan(**P42).forward(x).cpu().numpy().astype(np.float64)
    for i in range(len(X)):
        assert np.linalg.norm(a[i] - b[i]) <= 1e-5 * np.linalg.norm(a[i])


def test_forward_is_cuda_graph_capturable(jt):
    # jtfs_forward only enqueues work (the KD side stream joins through events), so a
    # CUDA graph capture replays the same bytes
    import torch
    kw = dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False)
    plan = jt.Plan(**kw)
    x = torch.from_numpy(signals.notes(5, N=2 ** 13, seed0=5)).cuda()
    out = torch.empty(5, plan.floats_per_signal, device="cuda")
    plan.forward(x, out)
    ref = out.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.forward(x, out)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.forward(x, out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_forward_host_buffers_and_batch_sharded_helper(jt):
    # jtfs_forward_host (the e2e entry point of bench.py: pinned host in / out, copies on
    # the stream) and shard.forward_batch_sharded (single process: no collective) give the
    # same bytes as jtfs_forward
    import torch
    from paper_2204_08269_b200 import shard
    plan = jt.Plan(**C1)
    X = np.concatenate([_c1_inputs(), signals.white(3, 2 ** 10, seed=21)]).astype(np.float32)
    x = torch.from_numpy(X).cuda()
    ref = plan.forward(x).cpu()
    xh = torch.from_numpy(X).pin_memory()
    oh = torch.empty(ref.shape, dtype=torch.float32).pin_memory()
    xd = torch.empty_like(x)
    od = torch.empty(ref.shape, dtype=torch.float32, device="cuda")
    plan.forward_host(xh, oh, xd, od)
    assert torch.equal(oh, ref)
    got = shard.forward_batch_sharded(plan, x).cpu()
    assert torch.equal(got, ref)
    assert shard.batch_slice(len(X), 1, 0) == (0, len(X))


# ---- joint stage alone (jtfs_debug_joint): stage parity and SURVEY §4 T4 invariants ----
def _y2_layout(s):
    """[(alpha, K, L, float offset)] of the tap-2 / debug_joint Y2 layout."""
    out, off = [], 0
    for a in s.alphas:
        K, L = len(s.adm[a]), s.N_pad >> s.k_alpha[a]
        out.append((a, K, L, off))
        off += 2 * K * L
    return out, off


def _pack_y2(s, Y2):
    lay, total = _y2_layout(s)
    flat = np.zeros(total, dtype=np.float32)
    for a, K, L, off in lay:
        blk = np.empty((2 * K, L), dtype=np.float32)
        blk[0::2] = Y2[a].real
        blk[1::2] = Y2[a].imag
        flat[off:off + 2 * K * L] = blk.ravel()
    return flat


def _random_y2(s, rng):
    Y2 = {}
    for a in s.alphas:
        K, L = len(s.adm[a]), s.N_pad >> s.k_alpha[a]
        scale = np.exp(rng.uniform(-2, 2, size=(K, 1)))        # rows of different magnitudes
        Y2[a] = ((rng.standard_normal((K, L)) + 1j * rng.standard_normal((K, L))) * scale)
        Y2[a] = Y2[a].astype(np.complex64).astype(np.complex128)
    Yphi = rng.standard_normal((s.n1, s.N_pad // s.p.T)).astype(np.float32).astype(np.float64)
    return Y2, Yphi


def _joint_gpu(jt, plan, s, Y2s, Yphis):
    import torch
    y2 = torch.from_numpy(np.stack([_pack_y2(s, Y2) for Y2 in Y2s])).cuda()
    yp = torch.from_numpy(np.stack([Yp.astype(np.float32).ravel() for Yp in Yphis])).cuda()
    out = plan.debug_joint(y2, yp)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("variant", ["eq3", "eq4"])
def test_joint_stage_parity_random_y2(jt, variant):
    # KD + KE against the oracle's joint stage (steps O7-O9) on random complex Y2 whose
    # rows span 4 decades -- stage-level parity independent of KA..KC
    kw = dict(C1, average_fr=(variant == "eq3"))
    prm = O.Params(**kw)
    s = O.schedule(prm)
    rng = np.random.default_rng(11)
    ins = [_random_y2(s, rng) for _ in range(3)]
    plan = jt.Plan(**kw)
    out = _joint_gpu(jt, plan, s, [y for y, _ in ins], [p for _, p in ins])
    for b, (Y2, Yphi) in enumerate(ins):
        maps = O.joint_stage(Y2, Yphi, s)
        _, _, s2 = plan.unpack(out[b])
        o = [maps[i] for i in range(len(s.paths))]
        e = path_errors(list(s2), o)
        assert e.max() <= TOL, (float(e.max()), int(np.argmax(e)))


@pytest.mark.parametrize("variant", ["eq3", "eq4"])
def test_joint_separable_grid_equal_spins(jt, variant):
    # T4: Y2_alpha[lambda][t] = a[lambda] b_alpha[t] with a REAL gives |psi_{beta,+1} *_lambda Y2|
    # = |psi_{beta,-1} *_lambda Y2| exactly (h_{+1} = conj h_{-1}, R10), so the two spins'
    # S2 maps of every (alpha, beta) coincide
    kw = dict(C1, average_fr=(variant == "eq3"))
    s = O.schedule(O.Params(**kw))
    rng = np.random.default_rng(5)
    a_prof = rng.standard_normal(s.n1)
    Y2 = {}
    for a in s.alphas:
        K, L = len(s.adm[a]), s.N_pad >> s.k_alpha[a]
        b = rng.standard_normal(L) + 1j * rng.standard_normal(L)
        Y2[a] = np.outer(a_prof[:K], b)
    Yphi = np.zeros((s.n1, s.N_pad // s.p.T))
    plan = jt.Plan(**kw)
    _, _, s2 = plan.unpack(_joint_gpu(jt, plan, s, [Y2], [Yphi])[0])
    paths = plan.paths()
    idx = {(k, th, a, b): i for i, (k, th, a, b, *_r) in enumerate(paths)}
    for (k, th, a, b), i in idx.items():
        if k == jt.PATH_SPIN and th == -1:
            j = idx[(k, +1, a, b)]
            ref = np.linalg.norm(s2[i]) + 1e-30
            assert np.linalg.norm(s2[i] - s2[j]) <= 1e-5 * ref, (a, b)


def test_joint_lambda_reversal_swaps_spins(jt):
    # T4: reversing the admissible rows, Y2'[lambda] = Y2[K-1-lambda], maps Z_theta(Y2')[r]
    # to Z_{-theta}(Y2)[K-1-r] on the circular lambda grid (h_theta[n] = h_{-theta}[-n], R9/R10);
    # Eq. (4) keeps every row at full rate, so S2'(theta)[r] = S2(-theta)[K-1-r], r < K
    kw = dict(C1, average_fr=False)
    s = O.schedule(O.Params(**kw))
    rng = np.random.default_rng(8)
    a0 = s.alphas[0]
    Y2, Y2r = {}, {}
    for a in s.alphas:
        K, L = len(s.adm[a]), s.N_pad >> s.k_alpha[a]
        Y2[a] = (rng.standard_normal((K, L)) + 1j * rng.standard_normal((K, L))) if a == a0 else np.zeros((K, L))
        Y2r[a] = Y2[a][::-1].copy()
    Yphi = np.zeros((s.n1, s.N_pad // s.p.T))
    plan = jt.Plan(**kw)
    out = _joint_gpu(jt, plan, s, [Y2, Y2r], [Yphi, Yphi])
    _, _, s2 = plan.unpack(out[0])
    _, _, s2r = plan.unpack(out[1])
    K = len(s.adm[a0])
    paths = plan.paths()
    idx = {(k, th, a, b): i for i, (k, th, a, b, *_r) in enumerate(paths)}
    checked = 0
    for (k, th, a, b), i in idx.items():
        if k == jt.PATH_SPIN and a == a0:
            j = idx[(k, -th, a, b)]
            got, ref = s2r[i][:K], s2[j][:K][::-1]
            assert np.linalg.norm(got - ref) <= 1e-5 * (np.linalg.norm(ref) + 1e-30), (th, b)
            checked += 1
    assert checked == 2 * plan.layout.n_beta


def test_c3_batch_independence_bench_launch(jt):
    # the bench's 256-signal launch (4 micro-batches of 64) gives each signal the same bytes
    # as a forward of that signal alone (per-signal work decomposition independent of B)
    import torch
    kw = dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4)
    plan = jt.Plan(**kw)
    X = torch.from_numpy(signals.notes(256, seed0=1000)).cuda()
    full = plan.forward(X)
    for b in (0, 1, 63, 64, 130, 255):
        one = plan.forward(X[b:b + 1].contiguous())
        assert torch.equal(full[b:b + 1].view(torch.int32), one.view(torch.int32)), b
