"""Multi-GPU ring on CPU: world_size-2 gloo processes replay the native
multi-GPU plan (hjb_exchange_plan -- the same code hjb_solve runs over NCCL)
with the oracle as each rank's step engine.  The result must equal the
single-process oracle bit for bit, which checks block ownership, the
per-step transfers (parallel.py:212-221, strategies.py:69-72) and the
per-sweep all-reduce (parallel.py:99-118, 239-244).  No GPU needed."""

import os
import socket

import numpy as np
import pytest

import oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, G, J, p, strategy, max_sweeps, out_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1008_4166_b200 import distributed as PD

    n = G.shape[1]
    nbl = 2 * p
    sizes = O.uniform_sizes(n, nbl)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    blocks = {b: np.asfortranarray(G[:, offs[b]:offs[b + 1]]).copy(order="F") for b in range(nbl)}
    Js = {b: np.ascontiguousarray(J[offs[b]:offs[b + 1]]) for b in range(nbl)}
    Ds = {b: O.column_norms2(blocks[b]) for b in range(nbl)}
    lo, hi = rank * p // world, (rank + 1) * p // world
    ring = O.RingSchedule(strategy, p)
    steps = O.steps_per_sweep(strategy, p)
    plan = PD.exchange_plan(strategy, p, world, rank, max_sweeps)
    sweeps_done, converged = 0, False
    for sweep in range(1, max_sweeps + 1):
        rot = 0
        for q in range(lo, hi):  # pre-pass on the blocks this GPU's workers hold
            for b in ring.layout()[q]:
                blocks[b - 1], Ds[b - 1], res = O.prepass_block(blocks[b - 1], Js[b - 1])
                rot += res[0]
        for s in range(steps):
            for q in range(lo, hi):
                i, j = ring.layout()[q]
                i, j = i - 1, j - 1
                blocks[i], blocks[j], Ds[i], Ds[j], res = O.pair_transform(
                    blocks[i], blocks[j], Ds[i], Ds[j], Js[i], Js[j])
                rot += res[0]
            ring.advance(sweep)
            reqs, recv = [], []
            for blk, peer, send in plan[(sweep - 1) * steps + s]:
                if send:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(blocks[blk].T)), peer))
                else:
                    buf = torch.empty((blocks[blk].shape[1], blocks[blk].shape[0]), dtype=torch.from_numpy(blocks[blk]).dtype)
                    reqs.append(dist.irecv(buf, peer))
                    recv.append((blk, buf))
            for r in reqs:
                r.wait()
            for blk, buf in recv:
                blocks[blk] = np.asfortranarray(buf.numpy().T)
                Ds[blk] = O.column_norms2(blocks[blk])
        t = torch.tensor([rot], dtype=torch.int64)
        dist.all_reduce(t)
        sweeps_done = sweep
        if int(t[0]) == 0:
            converged = True
            break
    # reassemble from the NATIVE final owner map (hjb_block_owners, what
    # hjb_solve gathers from), checked against this rank's replayed layout
    owners = PD.block_owners(strategy, p, world, sweeps_done)
    held = sorted(b - 1 for q in range(lo, hi) for b in ring.layout()[q])
    assert held == [b for b in range(nbl) if owners[b] == rank], (held, owners)
    out_q.put((rank, {b: blocks[b] for b in held}, sweeps_done, converged))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cplx,strategy,p,max_sweeps", [(False, "round_robin", 4, 30), (True, "modulus", 3, 30),
                                                        (False, "round_robin", 4, 3), (True, "modulus", 4, 2)])
def test_two_rank_ring_matches_single_process(cplx, strategy, p, max_sweeps):
    import torch.multiprocessing as mp

    rng = np.random.default_rng(11)
    n = 8 * p
    G = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    G = np.asfortranarray(G)
    J = np.array([1] * (n - n // 3) + [-1] * (n // 3), np.int8)
    ref, info = O.parallel_jacobi_2f(G, J, p, strategy, sweep_limit=max_sweeps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, G, J, p, strategy, max_sweeps, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    sizes = O.uniform_sizes(n, 2 * p)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    Gout = np.empty_like(G)
    seen = set()
    for rank, blocks, sweeps, conv in got:
        assert sweeps == info.sweeps and conv == info.converged
        for b, B in blocks.items():
            Gout[:, offs[b]:offs[b + 1]] = B
            seen.add(b)
    assert seen == set(range(2 * p))
    assert np.array_equal(Gout, ref)


def test_exchange_plan_is_symmetric():
    """Every send of GPU a to GPU b at a step is a receive of b from a."""
    from paper_1008_4166_b200 import distributed as PD

    for strategy in ("round_robin", "modulus"):
        for p, world in ((8, 2), (16, 4), (16, 8), (64, 8), (7, 3)):
            plans = [PD.exchange_plan(strategy, p, world, r, 2) for r in range(world)]
            for s in range(len(plans[0])):
                sends = sorted((r, peer, blk) for r in range(world) for blk, peer, sd in plans[r][s] if sd)
                recvs = sorted((peer, r, blk) for r in range(world) for blk, peer, sd in plans[r][s] if not sd)
                assert sends == recvs
                # one block out and one in per GPU boundary
                assert all(len(plans[r][s]) <= 2 * max(1, p // world) for r in range(world))


def _replayed_owners(strategy, p, world, sweeps):
    ring = O.RingSchedule(strategy, p)
    for sw in range(1, sweeps + 1):
        for _ in range(O.steps_per_sweep(strategy, p)):
            ring.advance(sw)
    from paper_1008_4166_b200 import distributed as PD
    own = np.full(2 * p, -1)
    for q, (i, j) in enumerate(ring.layout()):
        own[i - 1] = own[j - 1] = PD.gpu_of_worker(p, world, q)
    return own


@pytest.mark.parametrize("strategy", ["round_robin", "modulus"])
def test_final_owner_map_odd_and_even_sweeps(strategy):
    """hjb_block_owners == the oracle's ring replayed through exactly the
    sweeps run (parallel.py:299-301).  Round 1 read the owners after all
    max_sweeps advances, which is wrong for every odd sweep count: the
    layout has period 2 sweeps."""
    from paper_1008_4166_b200 import distributed as PD

    for p, world in ((16, 2), (32, 2), (128, 8), (64, 4), (7, 3)):
        for sweeps in (0, 1, 2, 14, 15, 17, 30):
            got = PD.block_owners(strategy, p, world, sweeps)
            assert np.array_equal(got, _replayed_owners(strategy, p, world, sweeps)), (p, world, sweeps)
        # the round-1 bug: owners after max_sweeps (30) instead of the 15 run
        if p >= 16:
            assert not np.array_equal(PD.block_owners(strategy, p, world, 15),
                                      PD.block_owners(strategy, p, world, 30))
