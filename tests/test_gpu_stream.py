"""Online reconstruction (paper P:118-119, "continuously regularized", "new incoming data can be added at
any time"): depth maps in batches → incremental fusion → regulariser continued from the carried state.
Checked against the oracle chain with the same state hand-over, bit for bit."""
import numpy as np
import pytest
import torch

import oracle
from synth.depth import sphere_depth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_1604_03734_b200 import Reconstruction
    return Reconstruction


def _oracle_handover(x_old, state_old, x_new, f_new, W_new):
    """The state of the old blocks placed into the grown block list; new blocks start warm (u = ū = f, p = 0);
    Ω̄ voxels hold u = ū = f, p = 0 (vol_load_state's convention)."""
    key = lambda x: [tuple(r) for r in x.tolist()]
    pos = {k: i for i, k in enumerate(key(x_new))}
    rows = np.array([pos[k] for k in key(x_old)])
    u, ub, p = state_old
    U, UB = f_new.astype(np.float32).copy(), f_new.astype(np.float32).copy()
    P = np.zeros((3,) + f_new.shape, np.float32)
    U[rows], UB[rows], P[:, rows] = u, ub, p
    bar = W_new == 0
    U[bar], UB[bar] = f_new[bar], f_new[bar]
    P[:, bar] = 0
    return U, UB, P


def test_two_batches_match_oracle(R):
    ds = sphere_depth()
    I = ds.intr.numpy()
    prm = (ds.voxel, ds.mu, ds.max_range, ds.w_max)
    lam, eps = 1.0, 0.01
    rec = R(I, *prm, lam=lam, eps=eps)
    rec.integrate(ds.depth[:3].cuda(), ds.poses[:3].cuda()).regularise(25)
    n1 = rec.n_blocks
    rec.integrate(ds.depth[3:].cuda(), ds.poses[3:].cuda()).regularise(30)
    assert rec.n_blocks > n1
    u_gpu = rec.u().cpu().numpy()
    # oracle chain with the same hand-over
    x1, _, f1, W1 = oracle.fuse(ds.depth[:3], I, ds.poses[:3], *prm)
    tau = float(np.float32(1 / 12 ** 0.5))
    st1 = oracle.regularise(x1, f1, W1, lam, eps, tau, tau, 25, precision="f32")
    x2, _, f2, W2 = oracle.fuse_incremental((x1, f1, W1), ds.depth[3:], I, ds.poses[3:], *prm)
    U, UB, P = _oracle_handover(x1, st1, x2, f2, W2)
    u2, _, _ = oracle.regularise(x2, f2, W2, lam, eps, tau, tau, 30, precision="f32", state=(U, UB, P))
    assert np.array_equal(rec.xyz.cpu().numpy(), x2)
    assert np.array_equal(u_gpu, u2)
    T = rec.extract()
    assert T.shape[0] > 1000
