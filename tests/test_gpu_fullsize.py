"""Full-size GPU parity at BASELINE.json's configurations, in the launch
configuration bench.py times (same plan cache, same nrhs widths).

* GPU vs the oracle's independent butterfly O2 on the same plan: the WHOLE
  output vector, relative l2 <= 1e-12 per column.
* GPU vs the dense sum O1 on sampled outputs the oracle computes one by one
  (rows for synthesis, modes for analysis): <= 10 x ID tolerance per column.

The plan is built once per box (GPU builder, ~3 min for configs[1]) into the
cache bench.py also uses.
"""
import os

import numpy as np
import pytest

import mht_inputs as mi
from paper_2605_21828_b200 import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def rel_cols(a, b):
    return max(np.linalg.norm(a[r] - b[r]) / np.linalg.norm(b[r]) for r in range(b.shape[0]))


def o2_err(a, b):
    """Per column, the larger of the relative l2 error and the elementwise
    max |a - b| / max |b| (every one of the n or m entries is compared)."""
    assert a.shape == b.shape
    return max(rel_cols(a, b), max(np.max(np.abs(a[r] - b[r])) / np.max(np.abs(b[r])) for r in range(b.shape[0])))


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a GPU")
    from paper_2605_21828_b200 import _build, mht

    _build.build()
    return mht


def _run(gpu, oracle_lib, w, dense_rows, dense_cols, drop_plan=False):
    path = W.ensure_plan(w, builder="gpu", log=None)
    torch.cuda.empty_cache()
    P = gpu.Plan(path)
    O = oracle_lib.Plan(path, verify_checksum=False)
    rng = np.random.default_rng(7)
    rows = np.sort(rng.choice(w.n, 1024, replace=False))
    cols = np.sort(rng.choice(w.m, 512, replace=False))
    for nrhs in w.nrhs:
        c = mi.workload_coefficients(w, nrhs)
        y = mi.workload_adjoint_input(w, nrhs)
        f = P.apply(torch.from_numpy(c).cuda()).cpu().numpy()
        a = P.adjoint(torch.from_numpy(y).cuda()).cpu().numpy()
        assert o2_err(f, O.apply(c)) <= 1e-12, ("fwd vs O2", nrhs)
        assert o2_err(a, O.adjoint(y)) <= 1e-12, ("adj vs O2", nrhs)
        sub = slice(0, min(nrhs, 4))  # a few columns against the (slow) dense sums
        fd = dense_rows(rows, c[sub])
        assert rel_cols(f[sub][:, rows], fd) <= 10 * w.tol, ("fwd vs dense", nrhs, rel_cols(f[sub][:, rows], fd))
        cd = dense_cols(cols, y[sub])
        assert rel_cols(a[sub][:, cols], cd) <= 10 * w.tol, ("adj vs dense", nrhs, rel_cols(a[sub][:, cols], cd))
    P.close()
    del O
    if drop_plan and not os.environ.get("MHT_KEEP_PLANS"):
        os.unlink(path)  # the plan cache lives in /dev/shm (host RAM): free it for the next workload


def test_config2_flat_65536_full_size(gpu, oracle_lib):
    """configs[1]: flat, n = m = 65,536, tol 1e-8, nrhs 1 and 32."""
    w = mi.WORKLOADS["c2"]
    x = mi.flat_points(w.n)
    k = mi.flat_workload_modes(w)
    _run(gpu, oracle_lib, w,
         lambda rows, c: oracle_lib.flat_synth(x[rows], k, c),
         lambda cols, y: oracle_lib.flat_analysis(x, k[cols], y))


def test_config2_quadtree_frequency_variant_full_size(gpu, oracle_lib):
    """NEXT-3: configs[1] with the 2-D kd (quadtree) frequency tree, nrhs 1 and 32."""
    w = mi.WORKLOADS["c2kd"]
    x = mi.flat_points(w.n)
    k = mi.flat_workload_modes(w)
    _run(gpu, oracle_lib, w,
         lambda rows, c: oracle_lib.flat_synth(x[rows], k, c),
         lambda cols, y: oracle_lib.flat_analysis(x, k[cols], y), drop_plan=True)


def test_config3_sphere_65536_full_size(gpu, oracle_lib):
    """configs[2]: sphere, n = m = 65,536 (l <= 255), tol 1e-10, nrhs 1 and 32."""
    w = mi.WORKLOADS["c3"]
    th, ph, _ = mi.sphere_points(w.n)
    lmax = w.extra["lmax"]

    def dense_cols(cols, y):
        full = oracle_lib.sphere_analysis(th, ph, lmax, y)   # all modes (one pass over the points)
        return full[:, cols]

    _run(gpu, oracle_lib, w,
         lambda rows, c: oracle_lib.sphere_synth(th[rows], ph[rows], lmax, c),
         dense_cols)


def test_config4_torus_mesh_full_size(gpu, oracle_lib):
    """configs[3]: torus mesh n = 32,768, m = 2,048 stored eigenvectors,
    Fiedler-tree rows, tol 1e-8, nrhs 1 and 64."""
    from mht_inputs import mesh as mm

    w = mi.WORKLOADS["c4"]
    _, _, _, Phi, _ = mm.torus_workload_inputs(w.extra["nu"], w.extra["nv"], w.m)
    _run(gpu, oracle_lib, w,
         lambda rows, c: oracle_lib.dense_synth(Phi[rows], c),
         lambda cols, y: oracle_lib.dense_analysis(Phi[:, cols], y))


@pytest.mark.skipif(os.environ.get("MHT_TEST_C5S") != "1",
                    reason="the c5 stand-in builds a ~100 GB plan (~10+ min); run with MHT_TEST_C5S=1 "
                           "(log committed under profiles/)")
def test_config5_standin_full_size(gpu, oracle_lib):
    """configs[4] stand-in (SURVEY.md §8(d) c5 protocol step 3; configs[4] itself,
    n = m = 2^20, probes to ~0.9 TB and 2^18 to 285 GB): flat n = m = 2^17 with the
    2^17 lowest eigenvalues, tol 1e-6, nrhs 1 and 16 — GPU vs O2 on the whole
    output, vs the dense sum on sampled rows / modes."""
    w = mi.WORKLOADS["c5s"]
    x = mi.flat_points(w.n)
    k = mi.flat_workload_modes(w)
    _run(gpu, oracle_lib, w,
         lambda rows, c: oracle_lib.flat_synth(x[rows], k, c),
         lambda cols, y: oracle_lib.flat_analysis(x, k[cols], y), drop_plan=not os.environ.get("MHT_KEEP_C5S"))
