"""N>1 host logic of the pipeline on CPU: two gloo ranks execute the engine's
own plan (ckf_pipeline_plan -- the op order every rank issues, including the
CheckFree+ swapped routes) with real send/recv, a toy fp64 stage function and
per-stage gradient accumulation in microbatch order.  The result must be
bit-identical to the single-rank run of the same plan, and every transfer must
pair up (a mismatch deadlocks -> the join timeout fails the test).

This is the multi-GPU path minus the device math: on a GPU box the same plan
is executed by Engine::move/hop with NCCL send/recv (tests/test_gpu_pipeline.py
checks on one GPU that the engine's transfers equal this plan)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

CASES = [
    # (stages, microbatches, swapped_half, placement, schedule); schedule 2 = 1F1B
    (4, 4, False, [0, 0, 1, 1], 1),
    (4, 4, True, [0, 0, 1, 1], 1),
    (4, 4, True, [0, 0, 1, 1], 0),
    (8, 6, True, [0, 0, 0, 0, 1, 1, 1, 1], 1),
    (8, 2, False, [0, 0, 0, 0, 1, 1, 1, 1], 0),
    (4, 8, False, [0, 0, 1, 1], 2),
    (4, 8, True, [0, 0, 1, 1], 2),
    (8, 16, True, [0, 0, 0, 0, 1, 1, 1, 1], 2),
    (4, 6, True, [0, 1, 0, 1], 2),  # interleaved placement: every route crosses the link 3x each way
    (4, 1, False, [0, 0, 1, 1], 2),  # a single microbatch
    (2, 3, False, [0, 1], 2),
]
# 4 ranks: one stage per rank (the swapped first/last-stage routes go 0 -> 1 -> 0 -> 2 -> 3 -> 2 -> 3)
CASES4 = [
    (4, 8, True, [0, 1, 2, 3], 2),
    (4, 8, False, [0, 1, 2, 3], 2),
    (8, 8, True, [0, 0, 1, 1, 2, 2, 3, 3], 2),
    (4, 4, True, [0, 1, 2, 3], 1),
]
N = 64  # toy activation width


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_plan(plan, s, m, me, xs, targets, params, send=None, recv=None):
    """Executes the ops of rank `me` in plan order.  Toy stage: h <- tanh(w_s h + b_s)."""
    w, b, e = params
    gw, gb, ge = np.zeros(s + 1), np.zeros(s + 1), 0.0
    h = {}
    cache = {}
    loss = {}
    for op in plan:
        k, kind = op["mb"], op["kind"]
        if kind == "xfer":
            if op["rank"] == me:
                send(h[k], op["arg"])
            elif op["arg"] == me:
                h[k] = recv(op["rank"])
            continue
        if op["rank"] != me:
            continue
        if kind == "embed_fwd":
            h[k] = xs[k] * e
        elif kind == "stage_fwd":
            sid = op["arg"]
            out = np.tanh(w[sid] * h[k] + b[sid])
            cache[(k, sid)] = (h[k], out)
            h[k] = out
        elif kind == "head":
            d = h[k] - targets[k]
            loss[k] = 0.5 * float(d @ d)
            h[k] = d  # from here on h[k] carries dL/dh
        elif kind == "stage_bwd":
            sid = op["arg"]
            inp, out = cache.pop((k, sid))
            da = h[k] * (1.0 - out * out)
            gw[sid] += float(da @ inp)
            gb[sid] += float(da.sum())
            h[k] = da * w[sid]
        elif kind == "embed_bwd":
            ge += float(h[k] @ xs[k])
    return gw, gb, ge, loss


def _inputs(s, m):
    rng = np.random.default_rng(7)
    xs = [rng.standard_normal(N) for _ in range(m)]
    ts = [rng.standard_normal(N) for _ in range(m)]
    params = (rng.standard_normal(s + 1) * 0.5, rng.standard_normal(s + 1) * 0.1, 0.7)
    return xs, ts, params


def _worker(rank, world, port, q, cases):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_15461_b200 import api
    results = []
    for (s, m, swapped, placement, schedule) in cases:
        plan = api.pipeline_plan(api.build_schedule(m, swapped, s), placement, schedule)
        xs, ts, params = _inputs(s, m)

        def send(arr, dst):
            dist.send(torch.from_numpy(np.ascontiguousarray(arr)), dst)

        def recv(src):
            t = torch.empty(N, dtype=torch.float64)
            dist.recv(t, src)
            return t.numpy()

        gw, gb, ge, loss = run_plan(plan, s, m, rank, xs, ts, params, send, recv)
        # stage grads live on their owners: gather everything to rank 0
        mine = np.array([1.0 if placement[i - 1] == rank else 0.0 for i in range(1, s + 1)])
        tw = torch.from_numpy(np.concatenate([gw[1:] * mine, gb[1:] * mine, [ge if rank == placement[0] else 0.0]]))
        dist.all_reduce(tw)
        ls = torch.tensor([loss.get(k, 0.0) for k in range(m)], dtype=torch.float64)
        dist.all_reduce(ls)
        results.append((tw.numpy().copy(), ls.numpy().copy(), sum(op["kind"] == "xfer" for op in plan)))
        dist.barrier()
    if rank == 0:
        q.put(results)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cases", [(2, CASES), (4, CASES4)])
def test_gloo_ranks_match_single_rank_bit_exactly(world, cases):
    from paper_2506_15461_b200 import api
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, cases)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (s, m, swapped, placement, schedule), (tw, ls, nx) in zip(cases, got):
        plan1 = api.pipeline_plan(api.build_schedule(m, swapped, s), [0] * s, schedule)
        assert not any(op["kind"] == "xfer" for op in plan1)
        xs, ts, params = _inputs(s, m)
        gw, gb, ge, loss = run_plan(plan1, s, m, 0, xs, ts, params)
        want = np.concatenate([gw[1:], gb[1:], [ge]])
        assert np.array_equal(tw, want), (s, m, swapped, schedule)
        assert np.array_equal(ls, [loss[k] for k in range(m)])
        # transfers: one boundary crossing per direction per microbatch, plus two more
        # per swapped microbatch when the swap straddles the rank boundary
        assert nx >= 2 * m


def test_plan_structure():
    from paper_2506_15461_b200 import api
    orders = api.build_schedule(4, True, 4)
    for schedule in (0, 1):
        plan = api.pipeline_plan(orders, [0, 0, 1, 1], schedule)
        # every stage runs forward and backward once per microbatch, on its owner
        for k in range(4):
            f = [op["arg"] for op in plan if op["mb"] == k and op["kind"] == "stage_fwd"]
            bwd = [op["arg"] for op in plan if op["mb"] == k and op["kind"] == "stage_bwd"]
            assert f == orders[k] and bwd == orders[k][::-1]
        for op in plan:
            if op["kind"] in ("stage_fwd", "stage_bwd"):
                assert op["rank"] == [0, 0, 1, 1][op["arg"] - 1]
        # GPipe: every forward precedes every backward; per-stage backward order = microbatch order
        if schedule == 1:
            last_f = max(i for i, op in enumerate(plan) if op["phase"] == 0)
            first_b = min(i for i, op in enumerate(plan) if op["phase"] == 1)
            assert last_f < first_b
        for sid in range(1, 5):
            mbs = [op["mb"] for op in plan if op["kind"] == "stage_bwd" and op["arg"] == sid]
            assert mbs == sorted(mbs)


def _check_1f1b(plan, orders, placement, m):
    """Structure of a schedule-2 plan: a topological order of the iteration; on every rank the
    stage backwards of each stage run in microbatch order (the reference's accumulation order)
    and at most `limit` microbatches are in flight; every transfer joins consecutive ops of one
    microbatch on different ranks."""
    from paper_2506_15461_b200 import api
    s = len(placement)
    limit = min(m, len(set(placement)))
    done = set()
    inflight = {r: set() for r in set(placement)}
    bwd_left = {}
    for r in set(placement):
        for k in range(m):
            bwd_left[(r, k)] = sum(1 for sid in orders[k] if placement[sid - 1] == r) + (1 if r == placement[0] else 0)
    last_bwd = {}
    for op in plan:
        k, kind = op["mb"], op["kind"]
        if kind == "xfer":
            continue
        r = op["rank"]
        # dependencies: forward route order, then head, then backward route order
        if kind == "stage_fwd":
            i = orders[k].index(op["arg"])
            assert ((k, "stage_fwd", orders[k][i - 1]) if i else (k, "embed_fwd", 0)) in done
        elif kind == "head":
            assert (k, "stage_fwd", orders[k][-1]) in done
        elif kind == "stage_bwd":
            i = orders[k].index(op["arg"])
            assert ((k, "stage_bwd", orders[k][i + 1]) if i < s - 1 else (k, "head", 0)) in done
            assert last_bwd.get(op["arg"], -1) < k  # per-stage accumulation in microbatch order
            last_bwd[op["arg"]] = k
        elif kind == "embed_bwd":
            assert (k, "stage_bwd", orders[k][0]) in done
        if kind in ("embed_fwd", "stage_fwd") and kind != "head":
            inflight[r].add(k)
            assert len(inflight[r]) <= limit, (r, inflight[r])
        if kind in ("stage_bwd", "embed_bwd"):
            bwd_left[(r, k)] -= 1
            if bwd_left[(r, k)] == 0:
                inflight[r].discard(k)
        done.add((k, kind, op["arg"] if kind.startswith("stage") else 0))
    assert len(done) == m * (2 * s + 3)


@pytest.mark.parametrize("s,m,placement", [(4, 8, [0, 0, 1, 1]), (8, 16, [0, 1, 2, 3, 4, 5, 6, 7]),
                                           (8, 64, [0, 1, 2, 3, 4, 5, 6, 7]), (4, 8, [0, 1, 2, 3]),
                                           (8, 12, [0, 0, 1, 1, 2, 2, 3, 3]), (4, 6, [0, 1, 0, 1]),
                                           # fewer microbatches than ranks, a single microbatch, one rank
                                           (4, 2, [0, 1, 2, 3]), (4, 1, [0, 1, 2, 3]), (4, 4, [0, 0, 0, 0]),
                                           (2, 3, [0, 1]), (6, 4, [0, 0, 0, 1, 1, 1])])
@pytest.mark.parametrize("swapped", [False, True])
def test_1f1b_plan_structure(s, m, placement, swapped):
    from paper_2506_15461_b200 import api
    if swapped and (s < 4 or m % 2):
        pytest.skip("swapped_half needs s >= 4 and an even microbatch count (pipeline.cpp:19-20, 50-51)")
    orders = api.build_schedule(m, swapped, s)
    plan = api.pipeline_plan(orders, placement, 2)
    _check_1f1b(plan, orders, placement, m)
    # the same transfers as GPipe (one per stage boundary crossing per direction), in another order
    x2 = sorted((o["mb"], o["rank"], o["arg"], o["aux"]) for o in plan if o["kind"] == "xfer")
    x1 = sorted((o["mb"], o["rank"], o["arg"], o["aux"]) for o in api.pipeline_plan(orders, placement, 1)
                if o["kind"] == "xfer")
    assert x1 == x2
