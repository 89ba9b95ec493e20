"""CPU fp64 restatement of the LLaMA-style stage block, its pipeline iteration and
its CheckFree / CheckFree+ trainer (torch autograd in float64 on the CPU).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Only tests/ and
oracle/make_llama_golden.py import this.

Parity status: the reference (/root/reference/proj) has no LLaMA block, so the
block ARITHMETIC is "parity unpinned" against it.  What
IS pinned is everything around it, reused from ckfree_oracle (checked against
the reference's own outputs in tests/test_oracle.py): counter RNG and init
streams (rng.hpp:10-48, model.cpp:27-33), stage partition (model.cpp:63-73),
schedules (pipeline.cpp:11-56), microbatch accumulation + Adam + omega
(pipeline.cpp:58-95, model.cpp:384-413), failure traces and the recovery /
trainer semantics (recovery.cpp:57-126, trainer.cpp:63-289).  The block itself
is validated with the reference's test METHODS (central finite differences,
tests/test_model.cpp:109-155) in tests/test_llama_oracle.py.

Block definition (mirrors paper_2506_15461_b200/csrc/llama_block.cu):
  h = E[tok];  per layer: h += attn(rope(RMSNorm(h; g1) Wqkv)) Wo;
                          h += (silu(g) * u) Wd with [g | u] = RMSNorm(h; g2) Wgu
  logits = RMSNorm(h; gF) E_inv;  loss = mean token cross-entropy.
  RMSNorm eps 1e-5; RoPE theta 1e4 on (j, j + hd/2) pairs, position = t mod T;
  causal softmax attention with scale 1/sqrt(hd).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from ckfree_oracle import (Adam, GOLDEN, _mix64_np, adam_update, build_schedule, bump_lr, counter_uniform,
                           derive_key, even_partition, parse_trace, recover_checkfree, standard_order,
                           sum_squares_fast, _w_or_u)

EPS = 1e-5
THETA = 10000.0


@dataclass
class LSpec:
    vocab: int
    d: int
    layers: int
    heads: int
    ffn: int
    seq_len: int
    stages: int

    @property
    def hd(self):
        return self.d // self.heads

    def layer_offsets(self):
        d, f = self.d, self.ffn
        o = {"g1": 0, "wqkv": d}
        o["wo"] = o["wqkv"] + 3 * d * d
        o["g2"] = o["wo"] + d * d
        o["wgu"] = o["g2"] + d
        o["wd"] = o["wgu"] + 2 * d * f
        o["total"] = o["wd"] + f * d
        return o

    def partition(self):
        return even_partition(self.layers, self.stages)

    @staticmethod
    def from_cfg(cfg: dict) -> "LSpec":
        return LSpec(int(cfg["vocab"]), int(cfg["model-dim"]), int(cfg["layers"]), int(cfg["heads"]),
                     int(cfg["hidden-dim"]), int(cfg["seq-len"]), int(cfg["stages"]))


# ------------------------------------------------------------------ token stream
def token_batch(data_seed: int, stream: int, index: int, rows: int, T: int, V: int) -> np.ndarray:
    """Counter-RNG sparse-bigram token process (csrc/tokens.cu), keyed like the
    reference's batches (dataset.cpp:15-20): key = derive_key(data_seed, stream, index).
    Integer-only -> bit-exact with the GPU generator."""
    key = derive_key(data_seed, stream, index)
    succ = np.uint64(derive_key(data_seed, 4))
    out = np.zeros((rows, T + 1), np.int64)
    r = np.arange(rows, dtype=np.uint64)
    prev = np.zeros(rows, np.uint64)
    Vu = np.uint64(V)
    with np.errstate(over="ignore"):
        for j in range(T + 1):
            c = r * np.uint64(T + 1) + np.uint64(j + 1)
            bits = _mix64_np(np.uint64(key) + c * np.uint64(GOLDEN))
            uni = ((bits & np.uint64(0xFFFFFFFF)) % Vu) * ((bits >> np.uint64(32)) % Vu) // Vu
            sel = (bits >> np.uint64(40)) & np.uint64(3)
            big = _mix64_np(succ ^ (np.uint64(4) * prev + sel)) % Vu
            first = (j == 0) | ((bits >> np.uint64(62)) == np.uint64(3))
            tok = np.where(first, uni, big)
            out[:, j] = tok.astype(np.int64)
            prev = tok
    return out.astype(np.int32)


# ------------------------------------------------------------------ init (fp32-rounded, like the GPU masters)
def _glorot(n, fan_in, fan_out, key):
    a = math.sqrt(6.0 / (fan_in + fan_out))
    return counter_uniform(key, -a, a, n).astype(np.float32).astype(np.float64)


def init_stage_flat(spec: LSpec, sid: int, seed: int) -> np.ndarray:
    o = spec.layer_offsets()
    first, last = spec.partition()[sid - 1]
    d, f = spec.d, spec.ffn
    out = []
    for l in range(first, last + 1):
        b = np.zeros(o["total"])
        b[o["g1"]:o["g1"] + d] = 1.0
        b[o["wqkv"]:o["wo"]] = _glorot(3 * d * d, d, 3 * d, derive_key(seed, 2 * l, 1))
        b[o["wo"]:o["g2"]] = _glorot(d * d, d, d, derive_key(seed, 2 * l, 2))
        b[o["g2"]:o["g2"] + d] = 1.0
        b[o["wgu"]:o["wd"]] = _glorot(2 * d * f, d, 2 * f, derive_key(seed, 2 * l + 1, 1))
        b[o["wd"]:o["total"]] = _glorot(f * d, f, d, derive_key(seed, 2 * l + 1, 2))
        out.append(b)
    return np.concatenate(out)


class LStage:
    def __init__(self, flat, lr):
        self.flat = flat
        self.opt = Adam.zeros(flat.size)
        self.omega = 0.0
        self.lr = lr


class LModel:
    def __init__(self, spec: LSpec, seed: int, lr: float):
        self.spec = spec
        self.stages = [LStage(init_stage_flat(spec, s, seed), lr) for s in range(1, spec.stages + 1)]
        self.embed = _glorot(spec.vocab * spec.d, spec.vocab, spec.d, derive_key(seed, 0))
        self.deembed = np.concatenate([np.ones(spec.d), _glorot(spec.d * spec.vocab, spec.d, spec.vocab,
                                                                 derive_key(seed, 1))])
        self.opt_embed = Adam.zeros(self.embed.size)
        self.opt_deembed = Adam.zeros(self.deembed.size)
        self.edge_lr = lr


# ------------------------------------------------------------------ block arithmetic (torch fp64)
def _rms(x, g):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + EPS) * g


def _rope(x, T):
    # x: [B, T, H, hd]
    hd = x.shape[-1]
    half = hd // 2
    j = torch.arange(half, dtype=torch.float64)
    inv = THETA ** (-2.0 * j / hd)
    ang = torch.arange(T, dtype=torch.float64)[:, None] * inv[None, :]
    c, s = torch.cos(ang)[None, :, None, :], torch.sin(ang)[None, :, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def _layer(h, W, spec: LSpec, B):
    d, f, H, hd, T = spec.d, spec.ffn, spec.heads, spec.hd, spec.seq_len
    o = spec.layer_offsets()
    g1 = W[o["g1"]:o["g1"] + d]
    Wqkv = W[o["wqkv"]:o["wo"]].view(d, 3 * d)
    Wo = W[o["wo"]:o["g2"]].view(d, d)
    g2 = W[o["g2"]:o["g2"] + d]
    Wgu = W[o["wgu"]:o["wd"]].view(d, 2 * f)
    Wd = W[o["wd"]:o["total"]].view(f, d)
    qkv = _rms(h, g1) @ Wqkv
    q, k, v = (qkv[:, i * d:(i + 1) * d].reshape(B, T, H, hd) for i in range(3))
    q, k = _rope(q, T), _rope(k, T)
    s = torch.einsum("bqhd,bkhd->bhqk", q, k) / math.sqrt(hd)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool), 1)
    s = s.masked_fill(mask, float("-inf"))
    p = torch.softmax(s, dim=-1)
    att = torch.einsum("bhqk,bkhd->bqhd", p, v).reshape(B * T, d)
    h = h + att @ Wo
    gu = _rms(h, g2) @ Wgu
    a = torch.nn.functional.silu(gu[:, :f]) * gu[:, f:]
    return h + a @ Wd


def microbatch(model: LModel, order, toks: np.ndarray, grad: bool = True, layer_mask=None):
    """forward (+ backward) of one microbatch along `order` (model.cpp:211-378 structure).
    Returns (loss, stage grads, embed grad, deembed grad)."""
    spec = model.spec
    d, V, T = spec.d, spec.vocab, spec.seq_len
    B = toks.shape[0]
    x = torch.as_tensor(toks[:, :T].reshape(-1), dtype=torch.long)
    y = torch.as_tensor(toks[:, 1:].reshape(-1), dtype=torch.long)
    Ws = [torch.tensor(s.flat, dtype=torch.float64, requires_grad=grad) for s in model.stages]
    E = torch.tensor(model.embed, dtype=torch.float64, requires_grad=grad)
    De = torch.tensor(model.deembed, dtype=torch.float64, requires_grad=grad)
    o = spec.layer_offsets()
    part = spec.partition()
    h = E.view(V, d)[x]
    for sid in order:
        first, last = part[sid - 1]
        W = Ws[sid - 1]
        for li in range(last - first + 1):
            h = _layer(h, W[li * o["total"]:(li + 1) * o["total"]], spec, B)
    logits = _rms(h, De[:d]) @ De[d:].view(d, V)
    loss = torch.nn.functional.cross_entropy(logits, y)
    if not grad:
        return float(loss), None, None, None
    loss.backward()
    return float(loss.detach()), [w.grad.numpy().copy() for w in Ws], E.grad.numpy().copy(), De.grad.numpy().copy()


def eval_loss(model: LModel, order, toks):
    with torch.no_grad():
        return microbatch(model, order, toks, grad=False)[0]


def accumulate_grads(model: LModel, orders, toks):
    """Sum of microbatch gradients in k order and the mean loss (pipeline.cpp:66-83)."""
    m = len(orders)
    rows = toks.shape[0]
    if rows == 0 or rows % m:
        raise ValueError("batch size must be divisible by the microbatch count")
    mb = rows // m
    tot_l, tot_s, tot_e, tot_d = 0.0, [np.zeros_like(s.flat) for s in model.stages], 0.0, 0.0
    for k in range(m):
        l, gs, ge, gd = microbatch(model, orders[k], toks[k * mb:(k + 1) * mb])
        tot_l += l
        tot_s = [a + b for a, b in zip(tot_s, gs)]
        tot_e = tot_e + ge
        tot_d = tot_d + gd
    return tot_l, tot_s, tot_e, tot_d


def run_iteration(model: LModel, orders, toks):
    """pipeline.cpp:58-95 on the LLaMA block: sum in k order, x 1/m, Adam per stage + omega, edges."""
    m = len(orders)
    tot_l, tot_s, tot_e, tot_d = accumulate_grads(model, orders, toks)
    inv = 1.0 / m
    for st, g in zip(model.stages, tot_s):
        g = g * inv
        st.opt.step += 1
        st.flat, st.opt.m, st.opt.v = adam_update(st.flat, st.opt.m, st.opt.v, g, st.lr, st.opt.step)
        st.omega = sum_squares_fast(g)
    model.opt_embed.step += 1
    model.embed, model.opt_embed.m, model.opt_embed.v = adam_update(
        model.embed, model.opt_embed.m, model.opt_embed.v, tot_e * inv, model.edge_lr, model.opt_embed.step)
    model.opt_deembed.step += 1
    model.deembed, model.opt_deembed.m, model.opt_deembed.v = adam_update(
        model.deembed, model.opt_deembed.m, model.opt_deembed.v, tot_d * inv, model.edge_lr, model.opt_deembed.step)
    return tot_l * inv, [s.omega for s in model.stages]


# ------------------------------------------------------------------ trainer (trainer.cpp:63-289)
def run_experiment(cfg: dict, trace_text: str, seed: int):
    """CheckFree / CheckFree+ / no-failures trainer on the LLaMA block.  Returns
    (evals[(iter, train, val)], events[(iter, stage, action, reduction_error, loss_spike)], unrecoverable)."""
    spec = LSpec.from_cfg(cfg)
    kind = cfg.get("strategy", "no-failures")
    iters = int(cfg.get("iters", 100))
    batch = int(cfg.get("batch", 32))
    m = int(cfg.get("microbatches", 8))
    lr = float(cfg.get("lr", 3e-4))
    evint = int(cfg.get("eval-interval", 25))
    val_size = int(cfg.get("val-size", 8))
    lr_bump = float(cfg.get("lr-bump", 1.1))
    swap_from = int(cfg.get("swap-from", 0))
    sched_mode = cfg.get("schedule", "auto")
    swapped = sched_mode == "swapped-half" or (sched_mode == "auto" and kind == "checkfree-plus")
    s = spec.stages
    data_seed = derive_key(seed, 12)  # trainer.cpp:22-24
    model = LModel(spec, derive_key(seed, 11), lr)
    T, V = spec.seq_len, spec.vocab
    val = token_batch(data_seed, 2, 0, val_size, T, V)
    std_sched = build_schedule(m, False, s)
    sw_sched = build_schedule(m, True, s) if swapped else None
    _, _, _, _, events = parse_trace(trace_text)
    grouped: dict[int, list] = {}
    for it, st in events:
        grouped.setdefault(it, []).append(st)

    def val_loss():
        return eval_loss(model, standard_order(s), val)

    evals, evs = [], []
    last_train = eval_loss(model, standard_order(s), token_batch(data_seed, 1, 1, batch, T, V))
    evals.append((0, last_train, val_loss()))
    replica = (model.embed.copy(), model.deembed.copy()) if kind == "checkfree-plus" else None
    model_iter = 0
    unrecoverable = False
    slot = 0
    for slot in range(1, iters + 1):
        swap_now = swapped and slot > swap_from
        toks = token_batch(data_seed, 1, model_iter + 1, batch, T, V)
        last_train, _ = run_iteration(model, sw_sched if swap_now else std_sched, toks)
        model_iter += 1
        if kind == "checkfree-plus":
            replica = (model.embed.copy(), model.deembed.copy())
        if kind != "no-failures" and slot in grouped:
            stages = sorted(grouped[slot])
            if any(b == a + 1 for a, b in zip(stages, stages[1:])):
                evs += [(slot, st, "unrecoverable", 0.0, 0.0) for st in stages]
                unrecoverable = True
                evals.append((slot, last_train, val_loss()))
                break
            vpre = val_loss()
            first_ev = len(evs)
            for st in stages:
                failed = model.stages[st - 1]
                old = failed.flat.copy()
                if st == 1 or st == s:
                    if kind != "checkfree-plus":
                        evs.append((slot, st, "unsupported", 0.0, 0.0))
                        unrecoverable = True
                        break
                    nb = model.stages[1] if st == 1 else model.stages[s - 2]
                    failed.flat = nb.flat.copy()
                    if st == 1:
                        model.embed = replica[0].copy()
                        model.opt_embed = Adam.zeros(model.embed.size)
                    else:
                        model.deembed = replica[1].copy()
                        model.opt_deembed = Adam.zeros(model.deembed.size)
                    failed.opt = Adam.zeros(failed.flat.size)
                    action = "edge_copy"
                else:
                    prev, nxt = model.stages[st - 2], model.stages[st]
                    fresh, deg = recover_checkfree(prev.flat, nxt.flat, prev.omega, nxt.omega)
                    action = "uniform_avg_fallback" if deg else "checkfree_avg"
                    failed.flat = np.array(fresh, np.float64)
                    failed.opt = Adam.zeros(failed.flat.size)
                failed.lr = bump_lr(failed.lr, lr_bump)
                failed.omega = 0.0
                evs.append((slot, st, action, sum_squares_fast(old - failed.flat), 0.0))
            if unrecoverable:
                evals.append((slot, last_train, val_loss()))
                break
            vpost = val_loss()
            for i in range(first_ev, len(evs)):
                a, b, c, dd, _ = evs[i]
                evs[i] = (a, b, c, dd, vpost - vpre)
        if slot % evint == 0 or slot == iters:
            evals.append((slot, last_train, val_loss()))
    if not evals or evals[-1][0] != slot:
        evals.append((slot, last_train, val_loss()))
    return evals, evs, unrecoverable
