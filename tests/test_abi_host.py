"""CPU tests of the C-ABI library (no GPU): it loads, exports every symbol jtfs.h
declares, validates parameters, and its host-side plan (schedule, layout, path
order, filter generator) agrees with the independent oracle.  No compute calls."""
import os
import re

import numpy as np
import pytest

from oracle import jtfs_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def jt():
    from paper_2204_08269_b200 import build
    build.build()
    from paper_2204_08269_b200 import jtfs
    return jtfs


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "jtfs.h")).read()
    return sorted(set(re.findall(r"^JTFS_API\s+(?:jtfs_status|const char\*)\s+(jtfs_\w+)\s*\(", src, re.M)))


def test_exports_every_declared_symbol(jt):
    lib = jt.library()
    decl = _header_symbols()
    assert len(decl) >= 12
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(jt.EXPORTS) == decl


def hostplan(jt, **kw):
    return jt.Plan(device=-1, **kw)


CFGS = {
    "c1": dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8),
    "c2": dict(N=2 ** 13, J=8, Q=16, J_fr=4, T=2 ** 13, F=16, average_fr=False),
    "c3": dict(N=2 ** 16, J=12, Q=16, J_fr=5, T=2 ** 13, F=4),
    "c4": dict(N=2 ** 17, J=13, Q=16, J_fr=5, T=2 ** 13, F=4),
    "p42": dict(N=2 ** 16, J=13, Q=16, J_fr=6, T=2 ** 11, F=4),
}


@pytest.mark.parametrize("name", list(CFGS))
def test_layout_and_paths_match_oracle(jt, name):
    kw = CFGS[name]
    p = hostplan(jt, **kw)
    s = O.schedule(O.Params(**kw))
    L = p.layout
    assert (L.n1, L.n_frames, L.frame0, L.lambda_out, L.n_paths, L.N_pad, L.N_fr) == \
        (s.n1, s.n_frames, s.frame0, s.lam_out, len(s.paths), s.N_pad, s.N_fr)
    assert L.floats_per_signal == O.unpack_layout(s)["total"]
    assert [(k, th, a, b) for (k, th, a, b, _, _) in p.paths()] == list(s.paths)
    np.testing.assert_allclose(p.lambda_xi(), s.xi1, rtol=1e-15)


def test_paper_44_by_32(jt):
    L = hostplan(jt, **CFGS["p42"]).layout
    assert (L.lambda_out, L.n_frames) == (44, 32)


@pytest.mark.parametrize("bank", [1, 2, 3, 4, 5])
def test_plan_filters_equal_oracle_filters(jt, bank):
    kw = CFGS["c1"]
    p = hostplan(jt, **kw)
    s = O.schedule(O.Params(**kw))
    grids = [(s.N_pad, s.N_pad), (s.N_pad // 8, s.N_pad), (s.N_fr, s.N_fr)]
    if bank in (1, 2, 3):
        xi, sg = {1: (s.xi1, s.sigma1), 2: (s.xi2, s.sigma2), 3: (s.xif, s.sigmaf)}[bank]
        for i in range(len(xi)):
            for L, n in grids:
                a = np.array(p.debug_filter(bank, i, L, n))
                b = O.morlet_hat(xi[i], sg[i], L, n)
                np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-300)
                assert a[0] == 0.0
    else:
        sig = s.sigma_T if bank == 4 else s.sigma_F
        for L, n in grids:
            np.testing.assert_allclose(p.debug_filter(bank, 0, L, n), O.gauss_hat(sig, L, n), rtol=1e-13)


@pytest.mark.parametrize("bad", [
    dict(N=1000, J=6, Q=8, J_fr=3, T=64),          # N not pow2
    dict(N=1024, J=11, Q=8, J_fr=3, T=64),         # 2^J > N
    dict(N=1024, J=6, Q=8, J_fr=3, T=2048),        # T > N
    dict(N=1024, J=6, Q=8, J_fr=3, T=63),          # T not pow2
    dict(N=1024, J=6, Q=0, J_fr=3, T=64),          # Q < 1
    dict(N=1024, J=6, Q=8, J_fr=3, T=64, F=3),     # F not pow2
    dict(N=1024, J=6, Q=8, J_fr=0, T=64),          # J_fr < 1
    dict(N=1024, J=1, Q=1, J_fr=3, T=64),          # n1 < 4
    dict(N=1024, J=6, Q=8, J_fr=3, T=64, F=1024),  # F > N_fr
])
def test_invalid_params_rejected(jt, bad):
    with pytest.raises(jt.JTFSError) as e:
        hostplan(jt, **bad)
    assert e.value.status == jt.JTFS_ERR_INVALID_ARG
    assert jt.library().jtfs_last_error()


def test_host_plan_refuses_forward_and_destroy_null(jt):
    import ctypes as C
    lib = jt.library()
    assert lib.jtfs_plan_destroy(None) == 0
    p = hostplan(jt, **CFGS["c1"])
    st = lib.jtfs_forward(p.handle, None, 0, None, None, 0, None)
    assert st == jt.JTFS_ERR_UNSUPPORTED    # host-only plans refuse every forward
    st = lib.jtfs_forward(p.handle, C.c_void_p(16), 1, C.c_void_p(16), C.c_void_p(256), 1 << 30, None)
    assert st == jt.JTFS_ERR_UNSUPPORTED
    assert p.workspace_size(8) > 0
    p.close()


# ---- second-order time scattering (Scattering1D) ----
SCAT1D = dict(N=2 ** 16, J=13, Q=16, J_fr=5, T=2 ** 11, F=4)   # the paper's setting


@pytest.mark.parametrize("kw", [dict(N=2 ** 10, J=6, Q=8, J_fr=3, T=2 ** 6, F=8), SCAT1D],
                         ids=["c1", "paper_s1d"])
def test_scat1d_layout_and_paths_match_oracle(jt, kw):
    plan = jt.Plan(**kw, device=-1)
    lay = plan.scat1d_layout
    s = O.schedule(O.Params(**kw))
    pairs = [(lam, a) for a in s.alphas for lam in s.adm[a]]
    assert lay.n1 == s.n1 and lay.n_frames == s.n_frames and lay.n2 == len(pairs)
    assert plan.scat1d_paths() == pairs
    assert lay.floats_per_signal == s.n_frames * (1 + s.n1 + len(pairs))


def test_scat1d_paper_shape(jt):
    # Q = 16, J = 13, T = 2^11 on the 2^16-sample excerpts -> 32 time frames,
    # first order n1 = 175 (the 1423-dim vector = n1 + n2; n2 depends on the
    # admissibility reading, so only n1 and the frames are pinned)
    lay = jt.Plan(**SCAT1D, device=-1).scat1d_layout
    assert (lay.n_frames, lay.n1) == (32, 175)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_u2_map_shape_matches_oracle(jt, name):
    # NEXT-4 scale-rate map (Fig. 1): host query vs the oracle's shape rule (reading R21)
    kw = CFGS[name]
    plan = hostplan(jt, **kw)
    s = O.schedule(O.Params(**kw))
    for pi, (kind, _, _, _) in enumerate(s.paths):
        if kind in (O.SPIN, O.PSI_T_PHI_F):
            assert plan.u2_map_shape(pi) == O.u2_map_shape(s, pi)
        else:
            with pytest.raises(jt.JTFSError):
                plan.u2_map_shape(pi)
    with pytest.raises(jt.JTFSError):
        plan.u2_map_shape(len(s.paths))


def test_library_reads_no_environment():
    # output bytes are a function of (plan params incl. flags, x) only: no source of the
    # library consults the process environment (env-dependent outputs)
    csrc = os.path.join(ROOT, "paper_2204_08269_b200", "csrc")
    for f in os.listdir(csrc):
        src = open(os.path.join(csrc, f)).read()
        assert "getenv" not in src, f


@pytest.mark.parametrize("name", list(CFGS))
def test_every_benchmarked_config_plans_on_the_tensor_cores(jt, name):
    # plan creation runs the tensor-core tiling (plan_tc); a config it cannot tile is an
    # explicit error unless JTFS_KD_SIMT is requested -- never a silent second backend
    p = hostplan(jt, **CFGS[name])
    assert p.floats_per_signal > 0
    q = hostplan(jt, **CFGS[name], flags=jt.JTFS_KD_SIMT)
    assert q.floats_per_signal == p.floats_per_signal


def test_a16_density_bookkeeping(jt):
    # jtfs_debug_a16_density on a host plan: per alpha the record / coefficient counts are
    # consistent, thresholds are monotone, and at thr = 0 every row's largest coefficient
    # (scaled into [2^13, 2^14)) makes its record live
    p = hostplan(jt, **CFGS["c1"])
    lay = p.layout
    d0, d1 = p.a16_density(0.0), p.a16_density(1e-3)
    assert len(d0) == lay.n_alpha
    for (tot, live, band, nkc, ent, coef), (tot1, live1, band1, _, ent1, coef1) in zip(d0, d1):
        assert tot == tot1 and coef == coef1 and tot % nkc == 0
        assert 0 < live <= band <= tot and 0 < ent <= coef
        assert live1 <= live and band1 <= band and ent1 <= ent
        assert live >= tot // nkc  # at least one live record per M-block


def test_kd_tiling_policy(jt):
    # the plan's KD tiling (jtfs_debug_kd_tiling) follows DESIGN.md §2: alpha 0 of c3 on
    # single CTAs with A stationary; CTA pairs (cta_group::2) on every other alpha when the
    # M-blocks split into pairs -- stationary where the A'' stream bounds the ring (10..15
    # K-chunks), a ring otherwise; JTFS_KD_NOPAIR disables pairs; odd block counts never pair
    t = hostplan(jt, **CFGS["c3"]).kd_tiling()
    assert all(a["kd_impl"] == 1 and a["Nt"] == 64 for a in t)
    assert (t[0]["pair"], t[0]["stat"]) == (0, 1)
    for a in t[1:]:
        assert a["pair"] == 1
        assert a["stat"] == (1 if 10 <= a["nkc"] < 16 else 0), a
        if a["stat"]:
            assert a["mblk"] == 1 and a["NBB"] >= 2
    assert not any(a["pair"] for a in hostplan(jt, **CFGS["c3"], flags=jt.JTFS_KD_NOPAIR).kd_tiling())
    for name in ("c2", "p42"):  # 5 / 11 M-blocks of 128 pair rows: no pairs
        assert not any(a["pair"] for a in hostplan(jt, **CFGS[name]).kd_tiling())
    assert all(a["kd_impl"] == 0 for a in hostplan(jt, **CFGS["c1"], flags=jt.JTFS_KD_SIMT).kd_tiling())
