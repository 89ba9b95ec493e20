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
    # (stages, microbatches, swapped_half, placement, schedule)
    (4, 4, False, [0, 0, 1, 1], 1),
    (4, 4, True, [0, 0, 1, 1], 1),
    (4, 4, True, [0, 0, 1, 1], 0),
    (8, 6, True, [0, 0, 0, 0, 1, 1, 1, 1], 1),
    (8, 2, False, [0, 0, 0, 0, 1, 1, 1, 1], 0),
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


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_15461_b200 import api
    results = []
    for (s, m, swapped, placement, schedule) in CASES:
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


def test_two_gloo_ranks_match_single_rank_bit_exactly():
    from paper_2506_15461_b200 import api
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (s, m, swapped, placement, schedule), (tw, ls, nx) in zip(CASES, got):
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
