"""Sharded plans: host-side exchange layout and the
multi-process all-to-all on CPU (gloo, world size 2 and 4), no GPU.

The layout from ``shard.exchange_sizes`` (computed from the plan file alone)
must partition z_ls exactly: every (tau, nu) block of the switch level goes
from the rank owning nu's frequency subtree to the rank owning tau's space
subtree, and the all-to-all with those split sizes delivers each block to its
owner in the order the receiver's loader lays them out.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import mht_inputs as mi
from paper_2605_21828_b200 import shard
from paper_2605_21828_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def plan_path(tmp_path_factory):
    d = tmp_path_factory.mktemp("shard")
    w = W.flat_workload(2048, 32, 4, 1e-8, name="shard")
    path = str(d / "shard.plan")
    W.build_workload_plan(w, path, workers=2, log=None)
    return path


@pytest.mark.parametrize("G", [1, 2, 4])
def test_exchange_layout_partitions_switch_level(plan_path, G):
    from paper_2605_21828_b200.precompute.planfile import PlanView

    pv = PlanView(plan_path)
    sizes, blocks, ls = shard.exchange_sizes(plan_path, G)
    nl = 1 << pv.L
    nf = nl >> ls
    r_out = pv.stages[ls].blocks["r_out"]
    # every block exactly once, total = all of z_ls
    seen = sorted(b for g in range(G) for h in range(G) for b in blocks[g][h])
    assert seen == [(t, v) for t in range(1 << ls) for v in range(nf)]
    assert sizes.sum() == int(np.sum(r_out))
    for g in range(G):
        for h in range(G):
            for t, v in blocks[g][h]:
                assert v // (nf // G) == g and t // ((1 << ls) // G) == h
    # balance: each rank sends and receives 1/G of the blocks
    assert all(len(sum((blocks[g][h] for h in range(G)), [])) == (1 << ls) * nf // G for g in range(G))


def test_switch_level_bounds():
    with pytest.raises(ValueError):
        shard.check_switch_level(4, 4, 1)
    with pytest.raises(ValueError):
        shard.check_switch_level(4, 3, 2)
    shard.check_switch_level(4, 4, 2)
    assert shard.default_switch_level(10, 8) == 5 and shard.default_switch_level(4, 4) == 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("G", [2, 4])
def test_all_to_all_delivers_blocks_gloo(plan_path, G, tmp_path):
    """G gloo ranks on CPU: rank g fills its send buffer with codes of the
    (tau, nu, entry) it owns, runs all_to_all_single with the layout's split
    sizes (forward), then sends the received codes back (the adjoint's reverse
    exchange); each rank checks it received exactly its space subtree's blocks
    in layout order, and got its own send buffer back."""
    script = tmp_path / "a2a.py"
    script.write_text(f'''
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {ROOT!r})
from paper_2605_21828_b200 import shard
from paper_2605_21828_b200.precompute.planfile import PlanView
dist.init_process_group("gloo")
g, G = dist.get_rank(), dist.get_world_size()
sizes, blocks, ls = shard.exchange_sizes({plan_path!r}, G)
pv = PlanView({plan_path!r})
nf = (1 << pv.L) >> ls
r_out = np.asarray(pv.stages[ls].blocks["r_out"])
def codes(bl):
    return np.concatenate([t * 10**9 + v * 10**4 + np.arange(r_out[t * nf + v]) for t, v in bl]) if bl else np.zeros(0)
send = torch.from_numpy(np.concatenate([codes(blocks[g][h]) for h in range(G)]).astype(np.float64))
recv = torch.empty(int(sizes[:, g].sum()), dtype=torch.float64)
dist.all_to_all_single(recv, send, output_split_sizes=[int(x) for x in sizes[:, g]],
                       input_split_sizes=[int(x) for x in sizes[g, :]])
want = np.concatenate([codes(blocks[src][g]) for src in range(G)])
assert np.array_equal(recv.numpy(), want), "forward exchange"
back = torch.empty_like(send)
dist.all_to_all_single(back, recv, output_split_sizes=[int(x) for x in sizes[g, :]],
                       input_split_sizes=[int(x) for x in sizes[:, g]])
assert torch.equal(back, send), "reverse exchange"
dist.barrier()
dist.destroy_process_group()
print("ok", g)
''')
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("ok") == G


@pytest.mark.parametrize("G", [2, 4])
def test_fused_exchange_host_tables_gloo(plan_path, G, tmp_path):
    """The fused exchange's host side on CPU (gloo): every rank lays out its
    workspace as the loader does (send regions destination by destination,
    receive regions source by source, after its own entries), exports
    (handle, layout) and all-gathers them with shard.gather_exports; then each
    rank stores its send blocks straight into the peers' receive buffers at
    send offset + (peer's receive offset for me - my send offset for the
    peer) — the delta mht_shard_set_peers gives the switch-stage kernels —
    and the reverse sums back the other way.  The buffers must equal what the
    all-to-all delivers, on every rank."""
    script = tmp_path / "fused.py"
    script.write_text(f'''
import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {ROOT!r})
from paper_2605_21828_b200 import shard
from paper_2605_21828_b200.precompute.planfile import PlanView
dist.init_process_group("gloo")
g, G = dist.get_rank(), dist.get_world_size()
sizes, blocks, ls = shard.exchange_sizes({plan_path!r}, G)
pv = PlanView({plan_path!r})
nf = (1 << pv.L) >> ls
r_out = np.asarray(pv.stages[ls].blocks["r_out"])
def codes(bl):
    return np.concatenate([t * 10**9 + v * 10**4 + np.arange(r_out[t * nf + v]) for t, v in bl]) if bl else np.zeros(0)
# rank-specific layout: some private entries first (a different amount per rank)
own = 1000 + 37 * g
send_off = own + np.concatenate([[0], np.cumsum(sizes[g, :])])[:G]
recv_base = own + int(sizes[g, :].sum()) + 11 * g
recv_off = recv_base + np.concatenate([[0], np.cumsum(sizes[:, g])])[:G]
Z = recv_base + int(sizes[:, g].sum())
layout = np.concatenate([recv_off, send_off, [8 * Z]]).astype(np.int64)
handles, lay = shard.gather_exports((bytes([g]) * shard.IPC_HANDLE_BYTES, layout), G)
assert lay.shape == (G, 2 * G + 1) and np.array_equal(lay[g], layout)
assert handles[g * 64:(g + 1) * 64] == bytes([g]) * 64
# every rank's workspace, as one object gathered (the "peer memory")
ws = np.full(Z, -1.0)
ws[send_off[0]:send_off[0] + sizes[g, :].sum()] = np.concatenate([codes(blocks[g][h]) for h in range(G)])
allws = [None] * G
dist.all_gather_object(allws, ws)
# forward: rank src's send block for h -> h's receive region, by the delta
for h in range(G):
    mine = allws[h].copy()
    for src in range(G):
        delta = lay[h][src] - lay[src][G + h]           # zdel[h] on rank src
        a = lay[src][G + h]
        n = int(sizes[src, h])
        mine[a + delta:a + delta + n] = allws[src][a:a + n]
    if h == g:
        want = np.concatenate([codes(blocks[src][g]) for src in range(G)])
        got = mine[recv_off[0]:recv_off[0] + sizes[:, g].sum()]
        assert np.array_equal(got, want), "fused forward delivery"
        fwd = mine
# reverse: rank g's receive region from src -> src's send region for g
allf = [None] * G
dist.all_gather_object(allf, fwd)
back = allws[g].copy()
back[send_off[0]:send_off[0] + sizes[g, :].sum()] = -2
for h in range(G):
    delta = lay[g][G + h] - lay[h][g]                    # zdel[G + g] on rank h
    a = lay[h][g]
    n = int(sizes[g, h])
    back[a + delta:a + delta + n] = allf[h][a:a + n]
assert np.array_equal(back, allws[g]), "fused reverse delivery"
dist.barrier()
dist.destroy_process_group()
print("ok", g)
''')
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("ok") == G
