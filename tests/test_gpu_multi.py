"""Multi-rank solve on real GPU pools: 2 ranks (gloo plumbing, pools on cuda:rank % ngpu) must
reproduce the single-GPU fixed-tree counts exactly while exchanging intervals -- over the native
peer-memory data plane (pbbgpu_group_*: CUDA IPC windows, device-side incumbent MIN, requests
and deposits; on a 1-GPU box both ranks share the device) and over the host-staged one."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import golden_io

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, name, ub, bound, split_mode, out, native=True, explorers=2048):
    import paper_2012_09511_b200 as pbb
    from paper_2012_09511_b200.multi import solve_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = rank % torch.cuda.device_count()
    pool = pbb.GpuPool(pbb.taillard_named(name), pbb.PoolConfig(device=dev, explorers=explorers, split_mode=split_mode),
                       bound=bound)
    res = solve_distributed(pool, ub, device="cpu", native=native)
    res2 = solve_distributed(pool, ub, device="cpu", native=native)   # the pool (and group) reused
    assert (res2.unique, res2.leaves) == (res.unique, res.leaves)
    out[rank] = (res.unique, res.leaves, res.best_value, res.remote_intervals, res.completed, res.hist)
    pool.close()
    dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("native", [True, False])
@pytest.mark.parametrize("name,ub,bound,split_mode", [("ta011", 1582, "lb1", 0), ("ta041", 2991, "lb1", 0),
                                                      ("ta011", 1582, "lb2", 0), ("ta041", 2991, "lb1", 1),
                                                      ("ta011", 1582, "lb2", 2)])
def test_two_ranks_match_single_gpu_counts(name, ub, bound, split_mode, native):
    gold = golden_io.ref_counts()[f"{name}@{ub}"] if bound == "lb1" else golden_io.lb2_counts()[f"{name}@{ub}"]
    want = gold["decomposed"] if bound == "lb1" else gold["unique"]
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, _port(), name, ub, bound, split_mode, out, native), nprocs=2,
                           start_method="spawn", join=True)
        r0, r1 = out[0], out[1]
    assert r0[0] == r1[0] == want
    assert r0[1] == r1[1] == gold["leaves"]
    assert r0[2] == r1[2] == ub
    assert r0[4] and r1[4]
    assert {str(k): v for k, v in r0[5].items()} == gold["hist"]


@pytest.mark.timeout(1200)
def test_two_ranks_native_ta021_lb2_exact_with_transfers():
    """The headline proof (ta021, LB2, UB 2297: 35,671,488 unique nodes) split over 2 ranks on the
    native peer-memory plane: exact count, and intervals did move between the ranks."""
    gold = golden_io.lb2_counts()["ta021@2297"]
    ctx = mp.get_context("spawn")
    moved = []
    # whether a rank runs dry while the other is still busy depends on how the two processes'
    # kernels interleave (on a 1-GPU box both ranks share the device): the count must be exact on
    # every attempt, and intervals must have moved on at least one of three
    for _ in range(3):
        with ctx.Manager() as mgr:
            out = mgr.dict()
            mp.start_processes(_worker, args=(2, _port(), "ta021", 2297, "lb2", 0, out, True, 0), nprocs=2,
                               start_method="spawn", join=True)
            r0, r1 = out[0], out[1]
        assert r0[0] == r1[0] == gold["unique"]
        assert r0[2] == r1[2] == 2297
        assert r0[3] == r1[3]
        moved.append(r0[3])
        if r0[3] > 0:
            break
    assert max(moved) > 0, moved


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,ub,bound", [("ta081", 6070, "lb1"), ("ta081", 6070, "lb2")])
def test_two_ranks_large_n_host_staged(name, ub, bound):
    """n > 64 explorer pools (int16 IVMs in HBM) on 2 ranks over the host-staged plane: the
    exported right halves (factoradic midpoints on the host) and the imports keep the
    fixed-tree count exact."""
    gold = golden_io.ref_counts()[f"{name}@{ub}"] if bound == "lb1" else golden_io.lb2_counts()[f"{name}@{ub}"]
    want = gold["decomposed"] if bound == "lb1" else gold["unique"]
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, _port(), name, ub, bound, 0, out, False, 1024), nprocs=2,
                           start_method="spawn", join=True)
        r0, r1 = out[0], out[1]
    assert r0[0] == r1[0] == want
    assert r0[1] == r1[1] == gold["leaves"]
    assert r0[2] == r1[2] == ub
    assert r0[4] and r1[4]
