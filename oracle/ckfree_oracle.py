"""CPU restatement of the reference's CheckFree / CheckFree+ hot path (numpy).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.

Parity status: PINNED.  Every function below is checked in
tests/test_oracle.py against tests/golden/*.json, which oracle/make_golden.py
produced by running the UNMODIFIED reference library (oracle/_ref, compiled
from /root/reference/proj/src).  Each function cites the reference file:line it
restates (paths relative to /root/reference/proj).
"""
from __future__ import annotations

import copy
import math
from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


# ---------------------------------------------------------------- rng.hpp:10-48
def mix64(x: int) -> int:
    """SplitMix64 finaliser (include/ckfree/rng.hpp:10-15)."""
    x = (x + GOLDEN) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def derive_key(seed: int, a: int = 0, b: int = 0, c: int = 0) -> int:
    """rng.hpp:18-25."""
    h = mix64(seed ^ 0x6A09E667F3BCC909)
    h = mix64(h ^ a)
    h = mix64(h ^ b)
    return mix64(h ^ c)


def to_unit(bits: int) -> float:
    """rng.hpp:28: upper 53 bits -> [0,1)."""
    return float(bits >> 11) * 2.0 ** -53


def unit_at(seed, a, b=0, c=0) -> float:
    return to_unit(derive_key(seed, a, b, c))


def _mix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(GOLDEN)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def counter_uniform(key: int, lo: float, hi: float, n: int, start: int = 0) -> np.ndarray:
    """CounterRng(key).uniform(lo,hi) draws start+1..start+n (rng.hpp:37-44).
    lo + (hi-lo)*u evaluated without FMA, exactly as the x86-64 reference."""
    ctr = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bits = _mix64_np(np.uint64(key) + ctr * np.uint64(GOLDEN))
    u = (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return lo + (hi - lo) * u


# ---------------------------------------------------------- failures.cpp:57-196
def hourly_to_per_iteration(p_hour: float, iter_s: float) -> float:
    """failures.cpp:57-61."""
    if not (0.0 <= p_hour < 1.0):
        raise ValueError("p_hour must lie in [0, 1)")
    if iter_s <= 0:
        raise ValueError("iteration_seconds must be positive")
    return 1.0 - math.pow(1.0 - p_hour, iter_s / 3600.0)


def generate_trace(seed: int, p_hour: float, iter_s: float, n_iters: int, stages) -> list[tuple[int, int]]:
    """failures.cpp:63-82: event iff unit_at(seed, iter, stage) < p_iter."""
    p = hourly_to_per_iteration(p_hour, iter_s)
    ev = []
    for it in range(1, n_iters + 1):
        for st in sorted(stages):
            if unit_at(seed, it, st) < p:
                ev.append((it, st))
    return ev


def _fmt17(v: float) -> str:
    s = "%.17g" % v
    return s


def serialize_trace(seed, p_hour, iter_s, stages, events) -> str:
    """failures.cpp:84-95 ('checkfree-trace v1')."""
    head = f"checkfree-trace v1 seed={seed} p_hour={_fmt17(p_hour)} iter_s={_fmt17(iter_s)} stages=" + \
        ",".join(str(s) for s in stages)
    return head + "\n" + "".join(f"{i},{s}\n" for i, s in events)


def parse_trace(text: str):
    """failures.cpp:97-155 -> (seed, p_hour, iter_s, stages, events)."""
    lines = text.split("\n")
    head = lines[0].split()
    if len(head) < 2 or head[0] != "checkfree-trace" or head[1] != "v1":
        raise ValueError("expected header 'checkfree-trace v1'")
    seed, p_hour, iter_s, stages = 0, 0.0, 3600.0, []
    for kv in head[2:]:
        k, _, v = kv.partition("=")
        if k == "seed":
            seed = int(v)
        elif k == "p_hour":
            p_hour = float(v)
        elif k == "iter_s":
            iter_s = float(v)
        elif k == "stages":
            stages = [int(t) for t in v.split(",") if t]
        else:
            raise ValueError(f"unknown header field '{k}'")
    events = []
    for ln in lines[1:]:
        if ln:
            a, b = ln.split(",")
            events.append((int(a), int(b)))
    return seed, p_hour, iter_s, stages, events


def consecutive_conflicts(events) -> list[tuple[int, int]]:
    """failures.cpp:171-184: lower stage of each adjacent pair dead in one iteration."""
    out = []
    by_iter: dict[int, set] = {}
    order = []
    for it, st in events:
        if it not in by_iter:
            by_iter[it] = set()
            order.append(it)
        by_iter[it].add(st)
    for it in order:
        s = by_iter[it]
        out += [(it, x) for x in sorted(s) if x + 1 in s]
    return out


def intermediate_stages(s):
    return list(range(2, s))   # failures.cpp:186-190


def all_stages(s):
    return list(range(1, s + 1))  # failures.cpp:192-196


# ------------------------------------------------------------- model.cpp:63-109
def even_partition(layers: int, stages: int) -> list[tuple[int, int]]:
    """model.cpp:63-73: first (L mod s) stages get one extra layer; 1-based inclusive."""
    out, nxt = [], 1
    for i in range(stages):
        cnt = layers // stages + (1 if i < layers % stages else 0)
        out.append((nxt, nxt + cnt - 1))
        nxt += cnt
    return out


# ---------------------------------------------------------- pipeline.cpp:11-56
def standard_order(s):
    return list(range(1, s + 1))


def swapped_order(s):
    """pipeline.cpp:18-26."""
    if s < 4:
        raise ValueError("swapped order requires at least 4 stages")
    o = standard_order(s)
    o[0], o[1] = o[1], o[0]
    o[s - 2], o[s - 1] = o[s - 1], o[s - 2]
    return o


def build_schedule(m: int, swapped_half: bool, s: int):
    """pipeline.cpp:41-56: swapped order at EVEN positions 0,2,4,..."""
    if m < 1:
        raise ValueError("microbatch count must be positive")
    if not swapped_half:
        return [standard_order(s) for _ in range(m)]
    if m % 2:
        raise ValueError("swapped_half schedule requires an even microbatch count")
    return [swapped_order(s) if k % 2 == 0 else standard_order(s) for k in range(m)]


# --------------------------------------------------------- recovery.cpp:57-126
def recover_checkfree(wp, wn, op: float, on: float):
    """recovery.cpp:57-73: (op*Wp + on*Wn)/(op+on); both zero -> uniform (degenerate)."""
    if op < 0 or on < 0:
        raise ValueError("gradient norms must be nonnegative")
    deg = False
    if op + on == 0.0:
        op = on = 1.0
        deg = True
    return (op * np.asarray(wp) + on * np.asarray(wn)) / (op + on), deg


def bump_lr(lr, factor):
    if lr <= 0:
        raise ValueError("learning rate must be positive")
    return factor * lr  # recovery.cpp:75-78


def reinit_uniform_avg(wp, wn):
    return 0.5 * (np.asarray(wp) + np.asarray(wn))  # recovery.cpp:105-110


def sum_squares(x) -> float:
    """kernels_serial.cpp:104-115: 1024-element block partials folded in order."""
    x = np.asarray(x, np.float64)
    total = 0.0
    for lo in range(0, x.size, 1024):
        blk = x[lo:lo + 1024]
        part = 0.0
        for v in blk:            # sequential inner sum, exactly as the reference
            part += v * v
        total += part
    return total


def sum_squares_fast(x) -> float:
    """Same reduction shape, vectorised inner sums (last-bit differences only)."""
    x = np.asarray(x, np.float64)
    total = 0.0
    for lo in range(0, x.size, 1024):
        total += float(np.dot(x[lo:lo + 1024], x[lo:lo + 1024]))
    return total


def reduction_error(wp, wf, wn, op, on):
    r, _ = recover_checkfree(wp, wn, op, on)
    return sum_squares_fast(r - np.asarray(wf))  # recovery.cpp:120-126


ADAM_B1, ADAM_B2, ADAM_EPS = 0.9, 0.999, 1e-8  # model.hpp:72-74


def adam_update(w, m, v, g, lr, step):
    """kernels_serial.cpp:133-144 (bias corrections with pow, no weight decay)."""
    bc1 = 1.0 - math.pow(ADAM_B1, step)
    bc2 = 1.0 - math.pow(ADAM_B2, step)
    m = ADAM_B1 * m + (1.0 - ADAM_B1) * g
    v = ADAM_B2 * v + (1.0 - ADAM_B2) * g * g
    w = w - lr * (m / bc1) / (np.sqrt(v / bc2) + ADAM_EPS)
    return w, m, v


# -------------------------------------------------------- model.cpp:159-413
@dataclass
class Spec:
    input_dim: int = 16
    hidden_dim: int = 64
    model_dim: int = 32
    output_dim: int = 16
    num_layers: int = 8
    num_stages: int = 4
    activation: str = "tanh"
    task: str = "regression"

    def partition(self):
        return even_partition(self.num_layers, self.num_stages)

    @staticmethod
    def from_cfg(cfg: dict) -> "Spec":
        return Spec(int(cfg.get("input-dim", 16)), int(cfg.get("hidden-dim", 64)), int(cfg.get("model-dim", 32)),
                    int(cfg.get("output-dim", 16)), int(cfg.get("layers", 8)), int(cfg.get("stages", 4)),
                    cfg.get("activation", "tanh"), cfg.get("task", "regression"))


@dataclass
class Adam:
    m: np.ndarray
    v: np.ndarray
    step: int = 0

    @staticmethod
    def zeros(n):
        return Adam(np.zeros(n), np.zeros(n), 0)

    def copy(self):
        return Adam(self.m.copy(), self.v.copy(), self.step)


@dataclass
class Stage:
    flat: np.ndarray          # blocks in order, [W1 (d x h) | W2 (h x d)] row-major (model.cpp:117-125)
    opt: Adam
    omega: float = 0.0
    lr: float = 3e-4


@dataclass
class Model:
    spec: Spec
    embed: np.ndarray         # [in x d]
    deembed: np.ndarray       # [d x out]
    opt_embed: Adam
    opt_deembed: Adam
    edge_lr: float
    stages: list = field(default_factory=list)

    def blocks(self, sid):
        """Views (W1, W2) of stage sid's blocks."""
        d, h = self.spec.model_dim, self.spec.hidden_dim
        f = self.stages[sid - 1].flat
        out, off = [], 0
        first, last = self.spec.partition()[sid - 1]
        for _ in range(first, last + 1):
            w1 = f[off:off + d * h].reshape(d, h)
            w2 = f[off + d * h:off + 2 * d * h].reshape(h, d)
            out.append((w1, w2))
            off += 2 * d * h
        return out

    def all_weights_flat(self):
        """model.cpp:145-157: embed, deembed, stages."""
        return np.concatenate([self.embed.ravel(), self.deembed.ravel()] + [s.flat for s in self.stages])

    def copy(self):
        return Model(self.spec, self.embed.copy(), self.deembed.copy(), self.opt_embed.copy(),
                     self.opt_deembed.copy(), self.edge_lr,
                     [Stage(s.flat.copy(), s.opt.copy(), s.omega, s.lr) for s in self.stages])


def sample_uniform(n, fan_in, fan_out, key):
    """model.cpp:27-33: U[-a,a], a = sqrt(6/(fan_in+fan_out))."""
    a = math.sqrt(6.0 / float(fan_in + fan_out))
    return counter_uniform(key, -a, a, n)


def init_stage_flat(spec: Spec, sid: int, seed: int) -> np.ndarray:
    """model.cpp:159-172: W1 tag 2l, W2 tag 2l+1 (1-based layer)."""
    d, h = spec.model_dim, spec.hidden_dim
    first, last = spec.partition()[sid - 1]
    parts = []
    for layer in range(first, last + 1):
        parts.append(sample_uniform(d * h, d, h, derive_key(seed, 2 * layer)))
        parts.append(sample_uniform(h * d, h, d, derive_key(seed, 2 * layer + 1)))
    return np.concatenate(parts)


def init_model(spec: Spec, seed: int, lr: float) -> Model:
    """model.cpp:174-197: embed tag 0, deembed tag 1."""
    e = sample_uniform(spec.input_dim * spec.model_dim, spec.input_dim, spec.model_dim, derive_key(seed, 0))
    de = sample_uniform(spec.model_dim * spec.output_dim, spec.model_dim, spec.output_dim, derive_key(seed, 1))
    m = Model(spec, e.reshape(spec.input_dim, spec.model_dim), de.reshape(spec.model_dim, spec.output_dim),
              Adam.zeros(e.size), Adam.zeros(de.size), lr)
    for sid in range(1, spec.num_stages + 1):
        f = init_stage_flat(spec, sid, seed)
        m.stages.append(Stage(f, Adam.zeros(f.size), 0.0, lr))
    return m


def _act(name, a):
    return np.tanh(a) if name == "tanh" else (np.maximum(a, 0.0) if name == "relu" else a.copy())


def _act_bwd(name, z, dz):
    if name == "tanh":
        return dz * (1.0 - z * z)
    if name == "relu":
        return np.where(z > 0.0, dz, 0.0)
    return dz.copy()


def forward(model: Model, order, x, layer_mask=None):
    """model.cpp:211-257 -> (predictions, cache)."""
    spec = model.spec
    h = x @ model.embed
    cache = []
    part = spec.partition()
    for sid in order:
        first, _ = part[sid - 1]
        for bi, (w1, w2) in enumerate(model.blocks(sid)):
            if layer_mask is not None and layer_mask[first + bi - 1] == 0:
                continue
            z = _act(spec.activation, h @ w1)
            cache.append((sid, bi, h.copy(), z))
            h = h + z @ w2
    pred = h @ model.deembed
    if not np.all(np.isfinite(pred)):
        raise FloatingPointError("forward: non-finite activation")
    return pred, (x, h, cache)


def prediction_grad(spec: Spec, pred, y):
    """model.cpp:260-275 (+ kernels_serial.cpp:146-185)."""
    rows, cols = pred.shape
    if spec.task == "regression":
        d = pred - y
        return float(np.sum(d * d)) / (rows * cols), 2.0 * d / (rows * cols)
    labels = y.astype(np.int64).ravel()
    mx = pred.max(axis=1, keepdims=True)
    ex = np.exp(pred - mx)
    den = ex.sum(axis=1, keepdims=True)
    loss = float(np.sum(-(pred[np.arange(rows), labels] - mx[:, 0] - np.log(den[:, 0])))) / rows
    p = ex / den
    p[np.arange(rows), labels] -= 1.0
    return loss, p / rows


def backward(model: Model, fwd, y):
    """model.cpp:314-378: returns (loss, g_stage[list of flat], g_embed, g_deembed)."""
    spec = model.spec
    pred, (x, h_final, cache) = fwd
    loss, dpred = prediction_grad(spec, pred, y)
    g_de = h_final.T @ dpred
    dh = dpred @ model.deembed.T
    g_st = [np.zeros_like(s.flat) for s in model.stages]
    d, hd = spec.model_dim, spec.hidden_dim
    for sid, bi, hin, z in reversed(cache):
        w1, w2 = model.blocks(sid)[bi]
        da = _act_bwd(spec.activation, z, dh @ w2.T)
        off = bi * 2 * d * hd
        g_st[sid - 1][off:off + d * hd] += (hin.T @ da).ravel()
        g_st[sid - 1][off + d * hd:off + 2 * d * hd] += (z.T @ dh).ravel()
        dh = dh + da @ w1.T
    g_e = x.T @ dh
    return loss, g_st, g_e, g_de


def adam_step_stage(st: Stage, g, lr):
    """model.cpp:384-397: step++, Adam, omega = ||g||^2."""
    st.opt.step += 1
    st.flat, st.opt.m, st.opt.v = adam_update(st.flat, st.opt.m, st.opt.v, g, lr, st.opt.step)
    st.omega = sum_squares_fast(g)


def run_iteration(model: Model, orders, x, y):
    """pipeline.cpp:58-95: contiguous microbatches, sum grads in k order, x 1/m, Adam per stage then edges."""
    m = len(orders)
    rows = x.shape[0]
    if rows == 0 or rows % m:
        raise ValueError("batch size must be divisible by the microbatch count")
    mb = rows // m
    tot_l, tot_s, tot_e, tot_d = 0.0, [np.zeros_like(s.flat) for s in model.stages], 0.0, 0.0
    for k in range(m):
        xs, ys = x[k * mb:(k + 1) * mb], y[k * mb:(k + 1) * mb]
        l, gs, ge, gd = backward(model, forward(model, orders[k], xs), ys)
        tot_l += l
        tot_s = [a + b for a, b in zip(tot_s, gs)]
        tot_e = tot_e + ge
        tot_d = tot_d + gd
    inv = 1.0 / m
    tot_s = [g * inv for g in tot_s]
    tot_e, tot_d, tot_l = tot_e * inv, tot_d * inv, tot_l * inv
    for st, g in zip(model.stages, tot_s):
        adam_step_stage(st, g, st.lr)
    model.opt_embed.step += 1
    e, model.opt_embed.m, model.opt_embed.v = adam_update(model.embed.ravel(), model.opt_embed.m, model.opt_embed.v,
                                                          tot_e.ravel(), model.edge_lr, model.opt_embed.step)
    model.embed = e.reshape(model.embed.shape)
    model.opt_deembed.step += 1
    de, model.opt_deembed.m, model.opt_deembed.v = adam_update(model.deembed.ravel(), model.opt_deembed.m,
                                                               model.opt_deembed.v, tot_d.ravel(), model.edge_lr,
                                                               model.opt_deembed.step)
    model.deembed = de.reshape(model.deembed.shape)
    return tot_l, [s.omega for s in model.stages]


# ------------------------------------------------------------ dataset.cpp:15-57
def make_batch(spec: Spec, teacher: Model, data_seed: int, stream: int, index: int, rows: int):
    """dataset.cpp:15-39: x ~ U[-1,1] keyed (data_seed, stream, index); y = teacher forward."""
    x = counter_uniform(derive_key(data_seed, stream, index), -1.0, 1.0, rows * spec.input_dim)
    x = x.reshape(rows, spec.input_dim)
    pred, _ = forward(teacher, standard_order(spec.num_stages), x)
    if spec.task == "regression":
        return x, pred
    return x, np.argmax(pred, axis=1).astype(np.float64).reshape(rows, 1)


class Task:
    """dataset.cpp:43-57 with the trainer's seeding (trainer.cpp:22-24)."""

    def __init__(self, spec: Spec, run_seed: int):
        self.spec = spec
        self.data_seed = derive_key(run_seed, 12)
        self.teacher = init_model(spec, derive_key(self.data_seed, 3), 1.0)

    def training_batch(self, model_iter, rows):
        return make_batch(self.spec, self.teacher, self.data_seed, 1, model_iter, rows)

    def validation_set(self, rows):
        return make_batch(self.spec, self.teacher, self.data_seed, 2, 0, rows)


# ------------------------------------------------------------- trainer.cpp:63-289
NEIGHBOR_KINDS = {"checkfree", "checkfree-plus", "reinit-random", "reinit-copy", "reinit-uniform-avg"}


def _w_or_u(wp, wn, a, b):
    if wp + wn == 0.0:
        return 0.5 * (a + b)
    return (wp * a + wn * b) / (wp + wn)  # trainer.cpp:33-36


def run_experiment(cfg: dict, trace_text: str, seed: int):
    """trainer.cpp:63-119 + handle_failures :146-289 for the neighbour family,
    no-failures, redundant and the checkpointing baseline (:173-193, checkpoint.cpp:70-83).  Returns (evals[(iter, train, val)],
    events[(iter, stage, action, reduction_error, loss_spike)], unrecoverable)."""
    spec = Spec.from_cfg(cfg)
    kind = cfg.get("strategy", "no-failures")
    iters = int(cfg.get("iters", 2000))
    batch = int(cfg.get("batch", 256))
    m = int(cfg.get("microbatches", 8))
    lr = float(cfg.get("lr", 3e-4))
    evint = int(cfg.get("eval-interval", 25))
    val_size = int(cfg.get("val-size", 1024))
    lr_bump = float(cfg.get("lr-bump", 1.1))
    averaged = cfg.get("recovered-moments", "fresh") == "averaged"
    swap_from = int(cfg.get("swap-from", 0))
    sched_mode = cfg.get("schedule", "auto")
    swapped = sched_mode == "swapped-half" or (sched_mode == "auto" and kind == "checkfree-plus")
    s = spec.num_stages

    task = Task(spec, seed)
    model = init_model(spec, derive_key(seed, 11), lr)
    vx, vy = task.validation_set(val_size)
    std_sched = build_schedule(m, False, s)
    sw_sched = build_schedule(m, True, s) if swapped else None
    _, _, _, _, events = parse_trace(trace_text)
    grouped: dict[int, list] = {}
    for it, st in events:
        grouped.setdefault(it, []).append(st)
    replica = None

    def val_loss():
        p, _ = forward(model, standard_order(s), vx)
        return prediction_grad(spec, p, vy)[0]

    evals, evs = [], []
    fx, fy = task.training_batch(1, batch)
    p, _ = forward(model, standard_order(s), fx)
    last_train = prediction_grad(spec, p, fy)[0]
    evals.append((0, last_train, val_loss()))
    if kind == "checkfree-plus":
        replica = (model.embed.copy(), model.deembed.copy())
    model_iter = 0
    ckpt_interval = int(cfg.get("checkpoint-interval", 100))
    snapshot = (copy.deepcopy(model), 0) if kind == "checkpointing" else None  # trainer.cpp:67-68
    unrecoverable = False
    slot = 0
    for slot in range(1, iters + 1):
        swap_now = swapped and slot > swap_from
        x, y = task.training_batch(model_iter + 1, batch)
        last_train, _ = run_iteration(model, sw_sched if swap_now else std_sched, x, y)
        model_iter += 1
        if kind == "checkfree-plus":
            replica = (model.embed.copy(), model.deembed.copy())
        if kind == "checkpointing" and model_iter % ckpt_interval == 0:  # trainer.cpp:83-85
            snapshot = (copy.deepcopy(model), model_iter)
        if kind == "checkpointing" and slot in grouped:
            # roll every stage back (adjacent failures included); data replays by model iteration
            stages = sorted(grouped[slot])
            vpre = val_loss()
            pre = [model.stages[st - 1].flat.copy() for st in stages]
            model = copy.deepcopy(snapshot[0])
            model_iter = snapshot[1]
            vpost = val_loss()
            evs += [(slot, st, "checkpoint_restore", sum_squares_fast(p0 - model.stages[st - 1].flat), vpost - vpre)
                    for st, p0 in zip(stages, pre)]
        elif kind != "no-failures" and slot in grouped:
            stages = sorted(grouped[slot])
            if any(b == a + 1 for a, b in zip(stages, stages[1:])):
                evs += [(slot, st, "unrecoverable", 0.0, 0.0) for st in stages]
                unrecoverable = True
                evals.append((slot, last_train, val_loss()))
                break
            if kind == "redundant":
                evs += [(slot, st, "redundant_copy", 0.0, 0.0) for st in stages]
            elif kind in NEIGHBOR_KINDS:
                vpre = val_loss()
                first_ev = len(evs)
                stop = False
                for st in stages:
                    failed = model.stages[st - 1]
                    old = failed.flat.copy()
                    if st == 1 or st == s:
                        if kind != "checkfree-plus":
                            evs.append((slot, st, "unsupported", 0.0, 0.0))
                            unrecoverable = True
                            stop = True
                            break
                        nb = model.stages[1] if st == 1 else model.stages[s - 2]
                        failed.flat = nb.flat.copy()
                        if st == 1:
                            model.embed = replica[0].copy()
                            model.opt_embed = Adam.zeros(model.embed.size)
                        else:
                            model.deembed = replica[1].copy()
                            model.opt_deembed = Adam.zeros(model.deembed.size)
                        failed.opt = nb.opt.copy() if averaged else Adam.zeros(failed.flat.size)
                        action = "edge_copy"
                    else:
                        prev, nxt = model.stages[st - 2], model.stages[st]
                        if kind in ("checkfree", "checkfree-plus"):
                            fresh, deg = recover_checkfree(prev.flat, nxt.flat, prev.omega, nxt.omega)
                            action = "uniform_avg_fallback" if deg else "checkfree_avg"
                        elif kind == "reinit-random":
                            fresh = init_stage_flat(spec, st, derive_key(seed, 13, slot, st))
                            action = "random_reinit"
                        elif kind == "reinit-copy":
                            fresh, action = prev.flat.copy(), "copy_prev"
                        else:
                            fresh, action = reinit_uniform_avg(prev.flat, nxt.flat), "uniform_avg"
                        failed.flat = np.array(fresh, np.float64)
                        if averaged and kind in ("checkfree", "checkfree-plus"):
                            failed.opt = Adam(_w_or_u(prev.omega, nxt.omega, prev.opt.m, nxt.opt.m),
                                              _w_or_u(prev.omega, nxt.omega, prev.opt.v, nxt.opt.v),
                                              min(prev.opt.step, nxt.opt.step))
                        else:
                            failed.opt = Adam.zeros(failed.flat.size)
                    failed.lr = bump_lr(failed.lr, lr_bump)
                    failed.omega = 0.0
                    evs.append((slot, st, action, sum_squares_fast(old - failed.flat), 0.0))
                if stop:
                    evals.append((slot, last_train, val_loss()))
                    break
                vpost = val_loss()
                for i in range(first_ev, len(evs)):
                    a, b, c, d, _ = evs[i]
                    evs[i] = (a, b, c, d, vpost - vpre)
        if slot % evint == 0 or slot == iters:
            evals.append((slot, last_train, val_loss()))
    if not evals or evals[-1][0] != slot:
        evals.append((slot, last_train, val_loss()))
    return evals, evs, unrecoverable


def parse_full_record(text: str):
    """Parses ref_run_experiment_full's E/F/U lines (oracle/ref_shim.cpp)."""
    evals, evs, unrec = [], [], False
    for ln in text.splitlines():
        p = ln.split(",")
        if p[0] == "E":
            evals.append((int(p[1]), float(p[2]), float(p[3])))
        elif p[0] == "F":
            evs.append((int(p[1]), int(p[2]), p[3], float(p[4]), float(p[5])))
        elif p[0] == "U":
            unrec = True
    return evals, evs, unrec
