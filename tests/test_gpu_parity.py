"""GPU parity: libmht (CUDA, through the C ABI) vs the oracle (CPU).

Bars (BASELINE.json north_star): relative l2 <= 1e-12 against the oracle's
independent butterfly apply O2 on the same plan, and <= 10 x the ID tolerance
against the dense sum O1, per column (reading A17).  Plans span several tiles
(64-row forward tiles, 32-column adjoint tiles) with ragged tails; edge cases
cover zero input, rank-0 / rank-1 matrices (COPY, alias and empty blocks),
ragged leaves, L = 0, multi-RHS widths that are not multiples of the register
blocking, the host-buffer API, determinism and corrupt plan files.
"""
import os

import numpy as np
import pytest

import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W
from paper_2605_21828_b200.precompute import build_plan, freq_tree, kd_tree
from paper_2605_21828_b200.precompute.basis import DenseBasis

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PARITY = 1e-12


def rel_cols(a, b):
    """max over columns of the relative l2 error (reading A17)."""
    a = np.atleast_2d(a)
    b = np.atleast_2d(b)
    out = []
    for r in range(a.shape[0]):
        nb = np.linalg.norm(b[r])
        out.append(np.linalg.norm(a[r] - b[r]) / (nb if nb > 0 else 1.0))
    return max(out)


def o2_err(a, b):
    """Parity against O2, element by element: per column, the larger of the
    relative l2 error and max_i |a_i - b_i| / max_i |b_i|.  One element off by
    more than 1e-12 of the column's scale fails, however long the column."""
    a = np.atleast_2d(a)
    b = np.atleast_2d(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    out = [rel_cols(a, b)]
    for r in range(a.shape[0]):
        mb = np.max(np.abs(b[r])) if b.shape[1] else 0.0
        out.append(np.max(np.abs(a[r] - b[r]), initial=0.0) / (mb if mb > 0 else 1.0))
    return max(out)


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    from paper_2605_21828_b200 import _build, mht

    _build.build()
    mht.load_library()
    return mht


@pytest.fixture(scope="module")
def plans(tmp_path_factory):
    return tmp_path_factory.mktemp("gpu_plans")


def flat_case(plans, n, side, L, tol, m=None, name="f"):
    w = W.flat_workload(n, side, L, tol, name=name)
    if m is not None:
        w = mi.Workload(name, "flat", n, m, "complex128", tol, L, (1,), {"side": side})
    path = str(plans / f"{name}_{n}_{side}_{L}_{tol:g}_{w.m}.plan")
    if not os.path.exists(path):
        W.build_workload_plan(w, path, workers=8, log=None)
    return path, w


def check_plan(gpu, oracle_lib, path, w, nrhs_list=(1,), dense=None):
    P = gpu.Plan(path)
    O = oracle_lib.Plan(path)
    for nrhs in nrhs_list:
        if w.dtype == "complex128":
            c = mi.complex_gaussian(nrhs, w.m, 100 + nrhs)
            y = mi.complex_gaussian(nrhs, w.n, 200 + nrhs)
        else:
            c = mi.real_gaussian(nrhs, w.m, 100 + nrhs)
            y = mi.real_gaussian(nrhs, w.n, 200 + nrhs)
        f = P.apply(torch.from_numpy(c).cuda()).cpu().numpy()
        ca = P.adjoint(torch.from_numpy(y).cuda()).cpu().numpy()
        assert o2_err(f, O.apply(c)) <= PARITY, ("fwd", nrhs)
        assert o2_err(ca, O.adjoint(y)) <= PARITY, ("adj", nrhs)
        if dense is not None:
            fd, cd = dense(c, y)
            assert rel_cols(f, fd) <= 10 * w.tol, ("fwd dense", nrhs, rel_cols(f, fd))
            assert rel_cols(ca, cd) <= 10 * w.tol, ("adj dense", nrhs, rel_cols(ca, cd))
    return P, O


def flat_dense(oracle_lib, w):
    x = mi.flat_points(w.n)
    k = mi.flat_workload_modes(w)
    return lambda c, y: (oracle_lib.flat_synth(x, k, c), oracle_lib.flat_analysis(x, k, y))


def test_flat_small_parity(gpu, oracle_lib, plans):
    path, w = flat_case(plans, 2048, 32, 4, 1e-8)
    check_plan(gpu, oracle_lib, path, w, (1, 2, 3, 5, 8, 16, 17, 32, 40), dense=flat_dense(oracle_lib, w))


def test_wide_rhs_blocks(gpu, oracle_lib, plans):
    """Wide right-hand-side blocks: nrhs 129 and 200 (several 32-column RHS
    chunks per tile plus a ragged last chunk, workspace strides above 128) on a
    complex flat plan and a real sphere plan, synthesis and analysis, element by
    element vs O2, plus the split into column blocks applied one by one (the
    transforms are column-independent; the blocks run other kernels — a single
    column takes the nrhs = 1 path — so they agree to 1e-12, not bitwise)."""
    path_c, wc = flat_case(plans, 2048, 32, 4, 1e-8)
    sp = str(plans / "sph_wide.plan")
    ws = W.sphere_workload(2048, 31, 4, 1e-10)
    W.build_workload_plan(ws, sp, workers=8, log=None)
    for path, w in ((path_c, wc), (sp, ws)):
        P, O = check_plan(gpu, oracle_lib, path, w, (129, 200))
        gen = mi.complex_gaussian if w.dtype == "complex128" else mi.real_gaussian
        c = torch.from_numpy(gen(129, w.m, 71)).cuda()
        f = P.apply(c)
        parts = torch.cat([P.apply(c[a:b].contiguous()) for a, b in ((0, 64), (64, 128), (128, 129))])
        assert o2_err(parts.cpu().numpy(), f.cpu().numpy()) <= PARITY
        P.close()


def test_flat_loose_tolerance_compressed(gpu, oracle_lib, plans):
    path, w = flat_case(plans, 4096, 32, 5, 1e-4)
    P, O = check_plan(gpu, oracle_lib, path, w, (1, 7), dense=flat_dense(oracle_lib, w))
    assert P.info.factor_entries < w.n * w.m


def test_config1_full_parity(gpu, oracle_lib, plans):
    """configs[0]: n = m = 4096, k in [-32,31]^2, tol 1e-8, nrhs 1, all rows."""
    w = mi.WORKLOADS["c1"]
    path = str(plans / "c1.plan")
    W.build_workload_plan(w, path, workers=8, log=None)
    check_plan(gpu, oracle_lib, path, w, (1, 4), dense=flat_dense(oracle_lib, w))


def test_config1_quadtree_frequency_variant(gpu, oracle_lib, plans):
    """NEXT-3 (§5): configs[0] with the frequency tree a 2-D
    kd tree over the frequency box (quadtree squares at even depths): full
    parity vs O2 element by element and vs the dense sum within 10 x tol."""
    w = mi.WORKLOADS["c1kd"]
    path = str(plans / "c1kd.plan")
    W.build_workload_plan(w, path, workers=8, log=None)
    check_plan(gpu, oracle_lib, path, w, (1, 4, 32), dense=flat_dense(oracle_lib, w))


def test_frequency_permutation_plan_paths(gpu, oracle_lib, plans):
    """A version-2 plan (perm_k: the quadtree-frequency order, c in the user's
    eigenvalue order, reading A18) through every path that reads or writes c:
    the nrhs = 1 kernels, the classic and
    warp-specialised DMMA kernels, the fused spectral filter on both sides and a
    2-way sharded emulation; all vs O2 element by element and vs the dense sum."""
    from paper_2605_21828_b200 import shard as SH

    w = mi.Workload("kdperm", "flat", 2048, 1024, "complex128", 1e-8, 4, (1,), {"side": 32, "ftree": "kd"})
    path = str(plans / "kdperm.plan")
    W.build_workload_plan(w, path, workers=8, log=None)
    P, O = check_plan(gpu, oracle_lib, path, w, (1, 5, 16, 33), dense=flat_dense(oracle_lib, w))
    c, y = mi.complex_gaussian(3, w.m, 7), mi.complex_gaussian(3, w.n, 8)
    ct, yt = torch.from_numpy(c).cuda(), torch.from_numpy(y).cuda()
    P.set_graphs(False)
    assert o2_err(P.apply(ct[:1]).cpu().numpy(), O.apply(c[:1])) <= PARITY
    assert o2_err(P.adjoint(yt[:1]).cpu().numpy(), O.adjoint(y[:1])) <= PARITY
    P.set_graphs(True)
    F = np.linspace(0.5, 2.0, w.m)
    Ft = torch.from_numpy(F).cuda()
    assert o2_err(P.apply_diag(ct, Ft).cpu().numpy(), O.apply(c * F[None, :])) <= PARITY
    assert o2_err(P.adjoint_diag(yt, Ft).cpu().numpy(), O.adjoint(y) * F[None, :]) <= PARITY
    P.close()
    shards = [SH.ShardPlan(path, 2, g, 0, -1) for g in range(2)]
    f = torch.zeros((3, w.n), dtype=torch.complex128, device="cuda")
    a = torch.zeros((3, w.m), dtype=torch.complex128, device="cuda")
    SH.emulate_apply(shards, ct, f)
    SH.emulate_adjoint(shards, yt, a)
    assert o2_err(f.cpu().numpy(), O.apply(c)) <= PARITY
    assert o2_err(a.cpu().numpy(), O.adjoint(y)) <= PARITY
    for sh in shards:
        sh.close()


def test_sphere_parity(gpu, oracle_lib, plans):
    lmax = 31
    w = W.sphere_workload(2048, lmax, 4, 1e-10)
    path = str(plans / "sph.plan")
    W.build_workload_plan(w, path, workers=8, log=None)
    th, ph, _ = mi.sphere_points(w.n)
    dense = lambda c, y: (oracle_lib.sphere_synth(th, ph, lmax, c), oracle_lib.sphere_analysis(th, ph, lmax, y))
    check_plan(gpu, oracle_lib, path, w, (1, 3, 16, 33, 64), dense=dense)


def test_ragged_leaves_and_L0(gpu, oracle_lib, plans):
    path, w = flat_case(plans, 1000, 32, 4, 1e-9, m=1000, name="ragged")
    check_plan(gpu, oracle_lib, path, w, (1, 3), dense=flat_dense(oracle_lib, w))
    path0, w0 = flat_case(plans, 64, 8, 0, 1e-12, name="L0")
    check_plan(gpu, oracle_lib, path0, w0, (1, 2), dense=flat_dense(oracle_lib, w0))


def test_full_rank_plan_identity_copy_paths(gpu, oracle_lib, plans):
    """tol ~ 0: many IDENTITY blocks -> alias and COPY resolution paths."""
    path, w = flat_case(plans, 1024, 32, 4, 1e-15, name="exact")
    P, _ = check_plan(gpu, oracle_lib, path, w, (1, 4, 32, 33), dense=flat_dense(oracle_lib, w))
    assert P.info.n_alias > 0


def _dense_plan(plans, Phi, L, tol, name):
    n, m = Phi.shape
    pts = np.random.default_rng(0).uniform(size=(n, 2))
    perm, sp_off = kd_tree(pts, L)
    path = str(plans / f"{name}.plan")
    build_plan(DenseBasis(Phi), perm, sp_off, freq_tree(m, L), L, tol, path, workers=1, log=None)
    return path


def test_rank0_rank1_and_exact_zero(gpu, oracle_lib, plans):
    rng = np.random.default_rng(4)
    u, v = rng.standard_normal(512), rng.standard_normal(512)
    w = mi.Workload("r1", "mesh", 512, 512, "float64", 1e-12, 3)
    p1 = _dense_plan(plans, np.outer(u, v), 3, 1e-12, "gpu_rank1")
    check_plan(gpu, oracle_lib, p1, w, (1, 5))
    p0 = _dense_plan(plans, np.zeros((512, 512)), 3, 1e-12, "gpu_rank0")
    P0 = gpu.Plan(p0)
    c = torch.from_numpy(rng.standard_normal((2, 512))).cuda()
    assert torch.count_nonzero(P0.apply(c)).item() == 0
    assert torch.count_nonzero(P0.adjoint(c)).item() == 0
    # c = 0 -> f = 0 exactly, and y = 0 -> 0
    path, wf = flat_case(plans, 2048, 32, 4, 1e-8)
    P = gpu.Plan(path)
    z = torch.zeros((1, wf.m), dtype=torch.complex128, device="cuda")
    assert torch.count_nonzero(P.apply(z)).item() == 0
    assert torch.count_nonzero(P.adjoint(torch.zeros((1, wf.n), dtype=torch.complex128, device="cuda"))).item() == 0


def test_determinism_and_host_api(gpu, oracle_lib, plans):
    path, w = flat_case(plans, 2048, 32, 4, 1e-8)
    P = gpu.Plan(path)
    c = mi.complex_gaussian(3, w.m, 9)
    y = mi.complex_gaussian(3, w.n, 10)
    ct = torch.from_numpy(c).cuda()
    yt = torch.from_numpy(y).cuda()
    f1, f2 = P.apply(ct), P.apply(ct)
    a1, a2 = P.adjoint(yt), P.adjoint(yt)
    assert torch.equal(f1, f2) and torch.equal(a1, a2)  # no atomics: bitwise deterministic
    fh = P.apply_host(c)
    ah = P.adjoint_host(y)
    assert np.array_equal(fh, f1.cpu().numpy()) and np.array_equal(ah, a1.cpu().numpy())
    # caller-supplied host outputs are checked before the C side writes into them
    for bad in (np.empty((3, w.n), dtype=np.float64), np.empty((3, w.n - 1), dtype=np.complex128),
                np.empty((w.n, 3), dtype=np.complex128).T):
        with pytest.raises(gpu.MhtError):
            P.apply_host(c, bad)
    ro = np.empty((3, w.m), dtype=np.complex128)
    ro.flags.writeable = False
    with pytest.raises(gpu.MhtError):
        P.adjoint_host(y, ro)
    out = np.empty((3, w.n), dtype=np.complex128)
    assert P.apply_host(c, out) is out and np.array_equal(out, fh)


def test_host_batch_pipelined(gpu, oracle_lib, plans):
    """mht_apply_host_batch (copies on the plan's copy streams overlapping the
    transforms, two staging slots): mixed synthesis / analysis jobs at several
    widths, more jobs than slots, pinned and pageable buffers, complex and real
    plans — bitwise equal to the device-buffer applies and to O2 element by
    element; two batches back to back; bad jobs rejected."""
    path_c, wc = flat_case(plans, 2048, 32, 4, 1e-8)
    sp = str(plans / "sph_batch.plan")
    ws = W.sphere_workload(2048, 31, 4, 1e-10)
    W.build_workload_plan(ws, sp, workers=8, log=None)
    for path, w in ((path_c, wc), (sp, ws)):
        P = gpu.Plan(path)
        O = oracle_lib.Plan(path)
        gen = mi.complex_gaussian if w.dtype == "complex128" else mi.real_gaussian
        jobs = [(0, gen(1, w.m, 601)), (1, gen(1, w.n, 602)), (0, gen(32, w.m, 603)), (1, gen(3, w.n, 604)),
                (0, gen(5, w.m, 605)), (1, gen(32, w.n, 606)), (0, gen(1, w.m, 607))]
        for rep in range(2):
            pinned = rep == 1
            jj = [(d, torch.from_numpy(x).pin_memory().numpy() if pinned else x) for d, x in jobs]
            outs = P.host_batch(jj)
            for (d, x), o in zip(jobs, outs):
                xt = torch.from_numpy(x).cuda()
                ref = (P.apply(xt) if d == 0 else P.adjoint(xt)).cpu().numpy()
                assert np.array_equal(o, ref), (path, d, x.shape, rep)
                assert o2_err(o, O.apply(x) if d == 0 else O.adjoint(x)) <= PARITY
        with pytest.raises(gpu.MhtError):
            P.host_batch_ptr([(2, 1, 1, 1)])
        with pytest.raises(gpu.MhtError):
            P.host_batch_ptr([(0, 0, 1, 1)])
        P.close()


def test_adjoint_identity_gpu(gpu, oracle_lib, plans):
    path, w = flat_case(plans, 2048, 32, 4, 1e-8)
    P = gpu.Plan(path)
    c = torch.from_numpy(mi.complex_gaussian(1, w.m, 1)).cuda()
    y = torch.from_numpy(mi.complex_gaussian(1, w.n, 2)).cuda()
    lhs = torch.vdot(y[0], P.apply(c)[0]).item()
    rhs = torch.vdot(P.adjoint(y)[0], c[0]).item()
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs) * 10


def test_corrupt_plan_rejected(gpu, plans):
    path, w = flat_case(plans, 2048, 32, 4, 1e-8)
    raw = bytearray(open(path, "rb").read())
    raw[len(raw) // 2] ^= 0x40
    bad = str(plans / "corrupt.plan")
    open(bad, "wb").write(raw)
    with pytest.raises(gpu.MhtError, match="FORMAT"):
        gpu.Plan(bad)
    with pytest.raises(gpu.MhtError, match="IO"):
        gpu.Plan(str(plans / "missing.plan"))
    P = gpu.Plan(path)
    with pytest.raises(gpu.MhtError):
        P.apply(torch.zeros((1, w.m + 1), dtype=torch.complex128, device="cuda"))


def test_cuda_graph_replay_matches_eager(gpu, plans):
    """Graph replay (default) and eager launches give bitwise-identical results,
    across repeated calls, new buffers and different widths."""
    import ctypes

    path, w = flat_case(plans, 2048, 32, 4, 1e-8)
    P = gpu.Plan(path)
    L = gpu.load_library()
    outs = {}
    for graphs in (1, 0):
        assert L.mht_set_graphs(ctypes.c_void_p(P._h), graphs) == 0
        for nrhs in (1, 5, 32):
            c = torch.from_numpy(mi.complex_gaussian(nrhs, w.m, 3)).cuda()
            y = torch.from_numpy(mi.complex_gaussian(nrhs, w.n, 4)).cuda()
            f = P.apply(c)
            f2 = P.apply(c)                      # replay
            a = P.adjoint(y, out=torch.empty_like(c))
            assert torch.equal(f, f2)
            outs[(graphs, nrhs)] = (f.cpu(), a.cpu())
    for nrhs in (1, 5, 32):
        assert torch.equal(outs[(1, nrhs)][0], outs[(0, nrhs)][0])
        assert torch.equal(outs[(1, nrhs)][1], outs[(0, nrhs)][1])


def test_forward_split_k_low_parallelism(gpu, oracle_lib, plans):
    """A stage with few row tiles and long rows takes the split-column path
    (partials + last-CTA fixup); results match O2 and stay bitwise
    deterministic across repeated applies."""
    rng = np.random.default_rng(11)
    n, m, L = 256, 4096, 2
    Phi = rng.standard_normal((n, m))
    path = _dense_plan(plans, Phi, L, 1e-12, "split_k")
    w = mi.Workload("sk", "mesh", n, m, "float64", 1e-12, L)
    P, O = check_plan(gpu, oracle_lib, path, w, (1, 3))
    c = torch.from_numpy(rng.standard_normal((1, m))).cuda()
    f1, f2 = P.apply(c), P.apply(c)
    assert torch.equal(f1, f2)
    fd = torch.from_numpy(Phi).cuda() @ c[0]
    assert (torch.linalg.vector_norm(f1[0] - fd) / torch.linalg.vector_norm(fd)).item() < 1e-11


def test_fused_group_sums_bitwise_equal_unfused(gpu, oracle_lib, plans):
    """Adjoint group sums formed on the consumer's load (default) and by the
    separate per-stage reduce pass give bitwise-identical results (same
    partials, same order), on a plan with aliases/COPY blocks (tol ~ 0), a
    compressed flat plan, and a real sphere plan; both match O2."""
    cases = [flat_case(plans, 1024, 32, 4, 1e-15, name="exact"), flat_case(plans, 2048, 32, 4, 1e-8)]
    lmax = 31
    ws = W.sphere_workload(2048, lmax, 4, 1e-10)
    sp = str(plans / "sph_fused.plan")
    W.build_workload_plan(ws, sp, workers=8, log=None)
    cases.append((sp, ws))
    for path, w in cases:
        P = gpu.Plan(path)
        O = oracle_lib.Plan(path)
        for nrhs in (1, 6, 32):
            if w.dtype == "complex128":
                y = mi.complex_gaussian(nrhs, w.n, 300 + nrhs)
            else:
                y = mi.real_gaussian(nrhs, w.n, 300 + nrhs)
            yt = torch.from_numpy(y).cuda()
            P.set_fused_sums(True)
            a1 = P.adjoint(yt).cpu()
            P.set_fused_sums(False)
            a0 = P.adjoint(yt).cpu()
            assert torch.equal(a1, a0), (path, nrhs)
            assert o2_err(a1.numpy(), O.adjoint(y)) <= PARITY
        P.set_fused_sums(True)
        P.close()


def test_split_k_small_blocks(gpu, oracle_lib, plans):
    """Few, short blocks (n_red 128..512) take the generalised split-column
    forward path (>= 64 columns per split), and few, tall blocks (1000+ rows)
    the split-row adjoint path (>= 128 rows per split), at nrhs = 1; parity vs
    O2 and the dense product, and bitwise determinism of both directions."""
    rng = np.random.default_rng(12)
    for n, m, L in ((128, 1024, 1), (512, 768, 2), (192, 2048, 3), (4096, 256, 2), (3000, 200, 1), (1001, 999, 2), (777, 333, 1)):
        Phi = rng.standard_normal((n, m))
        path = _dense_plan(plans, Phi, L, 1e-12, f"split_small_{n}_{m}_{L}")
        w = mi.Workload("sks", "mesh", n, m, "float64", 1e-12, L)
        P, _ = check_plan(gpu, oracle_lib, path, w, (1, 2, 17, 64))
        c = torch.from_numpy(rng.standard_normal((1, m))).cuda()
        f1, f2 = P.apply(c), P.apply(c)
        assert torch.equal(f1, f2)
        fd = torch.from_numpy(Phi).cuda() @ c[0]
        assert (torch.linalg.vector_norm(f1[0] - fd) / torch.linalg.vector_norm(fd)).item() < 1e-11
        y = torch.from_numpy(rng.standard_normal((1, n))).cuda()
        a1, a2 = P.adjoint(y), P.adjoint(y)
        assert torch.equal(a1, a2)
        ad = torch.from_numpy(Phi).cuda().T @ y[0]
        assert (torch.linalg.vector_norm(a1[0] - ad) / torch.linalg.vector_norm(ad)).item() < 1e-11
        P.close()


def test_multi_rhs_adjoint_k_split(gpu, oracle_lib, plans):
    """Tall blocks on a low-parallelism stage take the multi-RHS adjoint K
    split (row slabs summed in order by the last CTA): complex flat plan with
    n >> m, parity vs O2 and the dense sums at several widths, and bitwise
    determinism of repeated applies."""
    path, w = flat_case(plans, 8192, 16, 2, 1e-10, name="tall")
    P, _ = check_plan(gpu, oracle_lib, path, w, (2, 9, 32, 64), dense=flat_dense(oracle_lib, w))
    y = torch.from_numpy(mi.complex_gaussian(40, w.n, 77)).cuda()
    a1, a2 = P.adjoint(y), P.adjoint(y)
    assert torch.equal(a1, a2)
    P.close()


def test_applications_fused_diagonal(gpu, oracle_lib, plans):
    """PAPER.md §7: spectral filter f = Phi diag(F) c, filtered analysis
    diag(d) Phi^* f, GRF sample y = Phi sqrt(S) z and covariance product
    Phi S Phi^* v, each with the diagonal fused into the transform, against
    the oracle's O2 applied to the explicitly scaled vectors (plain
    definitions), at nrhs 1 and 5, complex and real plans, eager and graph."""
    path_c, wc = flat_case(plans, 2048, 32, 4, 1e-8)
    sp = str(plans / "sph_app.plan")
    ws = W.sphere_workload(2048, 31, 4, 1e-10)
    W.build_workload_plan(ws, sp, workers=8, log=None)
    rng = np.random.default_rng(31)
    for path, w in ((path_c, wc), (sp, ws)):
        P = gpu.Plan(path)
        O = oracle_lib.Plan(path)
        lam = np.sort(rng.uniform(0, 100, w.m))
        F = (lam < 40).astype(np.float64) + 0.5 * np.exp(-((lam - 70) / 10) ** 2)   # low-pass + bump (cf. Fig. 5)
        S = (1.0 + lam) ** -1.5                                                     # Matern-like spectral density
        Ft, St = torch.from_numpy(F).cuda(), torch.from_numpy(S).cuda()
        for graphs in (True, False):
            P.set_graphs(graphs)
            for nrhs in (1, 5):
                gen = mi.complex_gaussian if w.dtype == "complex128" else mi.real_gaussian
                c, y = gen(nrhs, w.m, 500 + nrhs), gen(nrhs, w.n, 600 + nrhs)
                ct, yt = torch.from_numpy(c).cuda(), torch.from_numpy(y).cuda()
                assert o2_err(P.apply_diag(ct, Ft).cpu().numpy(), O.apply(c * F[None, :])) <= PARITY
                assert o2_err(P.adjoint_diag(yt, Ft).cpu().numpy(), O.adjoint(y) * F[None, :]) <= PARITY
                assert o2_err(P.grf_sample(ct, St).cpu().numpy(), O.apply(c * np.sqrt(S)[None, :])) <= PARITY
                cov = O.apply(O.adjoint(y) * S[None, :])
                assert o2_err(P.covariance_apply(yt, St).cpu().numpy(), cov) <= PARITY
                # the plain transforms are unaffected afterwards (diagonal is per call)
                assert o2_err(P.apply(ct).cpu().numpy(), O.apply(c)) <= PARITY
        P.close()


def test_lsqr_inverse_mht(gpu, oracle_lib, plans):
    """Inverse MHT by LSQR (§7.1, Eq. inverse-MHT): the GPU LSQR (plan
    transforms + device vector kernels) follows the oracle's LSQR driven by
    O2 iterate by iterate (atol = btol = 0, same k), and converges to the
    dense least-squares solution; complex flat (n > m) and real mesh-like
    (random dense Phi) plans, nrhs 1 and 3."""
    from oracle.lsqr import lsqr_block

    w = W.flat_workload(1024, 16, 2, 1e-12, name="lsqr_gpu")
    path = str(plans / "lsqr_gpu.plan")
    W.build_workload_plan(w, path, workers=8, log=None)
    rng = np.random.default_rng(41)
    Phi_r = rng.standard_normal((600, 150))
    pr = _dense_plan(plans, Phi_r, 1, 1e-13, "lsqr_real")
    wr = mi.Workload("lr", "mesh", 600, 150, "float64", 1e-13, 1)
    x = mi.flat_points(w.n)
    k = mi.flat_modes(16)
    Phi_c = np.exp(1j * (x @ k.T.astype(float)))
    for path_, w_, Phi in ((path, w, Phi_c), (pr, wr, Phi_r)):
        P = gpu.Plan(path_)
        O = oracle_lib.Plan(path_)
        for nrhs in (1, 3):
            gen = mi.complex_gaussian if w_.dtype == "complex128" else mi.real_gaussian
            B = gen(nrhs, w_.n, 700 + nrhs)
            Bt = torch.from_numpy(B).cuda()
            for iters in (1, 4, 12):
                X, it, rn, an = P.lsqr(Bt, iters)
                assert it == iters
                Xo, rno, ano = lsqr_block(lambda v: O.apply(v[None, :])[0], lambda u: O.adjoint(u[None, :])[0], B, iters)
                assert rel_cols(X.cpu().numpy(), Xo) <= 1e-10, (path_, nrhs, iters)
                assert np.allclose(rn, rno, rtol=1e-9, atol=0)
            X, it, rn, an = P.lsqr(Bt, 400, atol=1e-12, btol=1e-12)
            assert it < 400
            Xs = np.linalg.lstsq(Phi, B.T, rcond=None)[0].T
            assert rel_cols(X.cpu().numpy(), Xs) <= 1e-8, (path_, nrhs, it)
        P.close()


def test_sharded_plan_emulated_on_one_gpu(gpu, oracle_lib, plans):
    """SURVEY §8(e) sharded plans: G = 2 and 4 shards of one plan (frequency
    subtrees for stages <= ls, space subtrees after, one all-to-all of z_ls),
    all loaded on this GPU with the exchange done by device copies, then with
    the fused exchange (switch-stage stores into the other shards' receive
    buffers and the reverse sums into their send buffers, arrival flags; two
    rounds of applies so the epochs advance).  The assembled synthesis and
    analysis match O2 on the whole plan (<= 1e-12) at nrhs 1, 5 and 32,
    complex flat and real sphere plans, every admissible switch level, the
    fused results bitwise those of the copy exchange; each shard holds about
    1/G of the factor bytes."""
    from paper_2605_21828_b200 import shard as SH

    path_c, wc = flat_case(plans, 2048, 32, 4, 1e-8)
    sp = str(plans / "sph_shard.plan")
    ws = W.sphere_workload(2048, 31, 4, 1e-10)
    W.build_workload_plan(ws, sp, workers=8, log=None)
    for path, w in ((path_c, wc), (sp, ws)):
        O = oracle_lib.Plan(path)
        full = gpu.Plan(path)
        total = full.info.factor_entries
        full.close()
        for G in (2, 4):
            lg = G.bit_length() - 1
            for ls in range(lg, w.L - lg + 1):
                shards = [SH.ShardPlan(path, G, g, 0, ls) for g in range(G)]
                assert all(s.ls == ls for s in shards)
                held = sum(s.info.factor_entries for s in shards)
                assert held == total                           # every block on exactly one rank
                assert max(s.info.factor_entries for s in shards) <= 0.75 * total if G == 4 else True
                res = {}
                for fused in (False, True):
                    if fused:
                        # the fused exchange: switch-stage stores straight into the
                        # other shards' receive buffers, arrival flags per apply
                        SH.emulate_fuse(shards, 32)
                    for rep in range(2 if fused else 1):
                        for nrhs in (1, 5, 32):
                            gen = mi.complex_gaussian if w.dtype == "complex128" else mi.real_gaussian
                            c, y = gen(nrhs, w.m, 800 + nrhs), gen(nrhs, w.n, 900 + nrhs)
                            ct, yt = torch.from_numpy(c).cuda(), torch.from_numpy(y).cuda()
                            f = torch.zeros((nrhs, w.n), dtype=shards[0].torch_dtype, device="cuda")
                            a = torch.zeros((nrhs, w.m), dtype=shards[0].torch_dtype, device="cuda")
                            SH.emulate_apply(shards, ct, f)
                            SH.emulate_adjoint(shards, yt, a)
                            assert o2_err(f.cpu().numpy(), O.apply(c)) <= PARITY, (path, G, ls, nrhs, fused)
                            assert o2_err(a.cpu().numpy(), O.adjoint(y)) <= PARITY, (path, G, ls, nrhs, fused)
                            if fused:  # same arithmetic, other store addresses: bitwise equal
                                assert torch.equal(f, res[nrhs][0]) and torch.equal(a, res[nrhs][1]), (G, ls, nrhs)
                            else:
                                res[nrhs] = (f, a)
                for s in shards:
                    s.unfuse()
                    s.close()


@pytest.mark.parametrize("family", ["sphere", "flat"])
def test_multi_rhs_kernels_repeatable(gpu, oracle_lib, plans, family):
    """The multi-RHS kernels at nrhs >= 32 (complex: warp-specialised TMA
    kernel; real: 16-byte cp.async ring kernel) and below (classic DMMA
    kernel, nrhs 17) on plans with several row tiles per block and K tails:
    12 repeated synthesis / analysis applies are bitwise identical (no race
    between the TMA / cp.async producers and the consumers) and match O2
    element by element."""
    if family == "sphere":
        w = W.sphere_workload(4096, 63, 6, 1e-10)
    else:
        w = W.flat_workload(4096, 64, 6, 1e-8, name="flat_rep")
    path = str(plans / f"{family}_rep.plan")
    if not os.path.exists(path):
        W.build_workload_plan(w, path, workers=8, log=None)
    P = gpu.Plan(path)
    P.set_graphs(False)
    O = oracle_lib.Plan(path)
    gen = mi.real_gaussian if w.dtype == "float64" else mi.complex_gaussian
    for nrhs in (17, 32, 40):
        c = gen(nrhs, w.m, 1000 + nrhs)
        y = gen(nrhs, w.n, 1100 + nrhs)
        ct, yt = torch.from_numpy(c).cuda(), torch.from_numpy(y).cuda()
        f0, a0 = P.apply(ct), P.adjoint(yt)
        for _ in range(12):
            assert torch.equal(P.apply(ct), f0) and torch.equal(P.adjoint(yt), a0)
        assert o2_err(f0.cpu().numpy(), O.apply(c)) <= PARITY
        assert o2_err(a0.cpu().numpy(), O.adjoint(y)) <= PARITY
    P.close()


def test_multi_rhs_stress_repeatable(gpu, oracle_lib, plans):
    """Race stress for the multi-RHS pipelines (compute-sanitizer is closed on
    this pool, profiles/r02_sanitizer_closed.txt): 60 back-to-back synthesis +
    analysis pairs per width on a complex plan (warp-specialised TMA / mbarrier
    kernel at nrhs >= 32, including a partial second RHS chunk, and the K-split
    slabs of tall blocks) and a real plan (cp.async ring kernel), graphs on, no
    synchronisation between applies; every result is bitwise identical to the
    first, which matches O2 element by element."""
    cases = [flat_case(plans, 8192, 16, 2, 1e-10, name="tall"), flat_case(plans, 2048, 32, 4, 1e-8)]
    sp = str(plans / "sph_stress.plan")
    ws = W.sphere_workload(2048, 31, 4, 1e-10)
    W.build_workload_plan(ws, sp, workers=8, log=None)
    cases.append((sp, ws))
    for path, w in cases:
        P = gpu.Plan(path)
        O = oracle_lib.Plan(path)
        gen = mi.real_gaussian if w.dtype == "float64" else mi.complex_gaussian
        for nrhs in (32, 48, 64):
            c, y = gen(nrhs, w.m, 1400 + nrhs), gen(nrhs, w.n, 1500 + nrhs)
            ct, yt = torch.from_numpy(c).cuda(), torch.from_numpy(y).cuda()
            f0, a0 = P.apply(ct).clone(), P.adjoint(yt).clone()
            fs, as_ = [], []
            for _ in range(60):
                fs.append(P.apply(ct).clone())
                as_.append(P.adjoint(yt).clone())
            torch.cuda.synchronize()
            assert all(torch.equal(f0, x) for x in fs) and all(torch.equal(a0, x) for x in as_), (path, nrhs)
            assert o2_err(f0.cpu().numpy(), O.apply(c)) <= PARITY
            assert o2_err(a0.cpu().numpy(), O.adjoint(y)) <= PARITY
        P.close()
