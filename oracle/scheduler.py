"""oracle/scheduler.py -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Plain-Python reference of NEO's load-aware scheduler (Sec 3.2,
P:250-291), written step by step in the paper's order and notation, used to
check the native implementation (neo_schedule in libneo) decision by decision.
Readings where the paper is silent are DESIGN.md s1-s8 (shared with the native
code's header, include/neo.h).

Cost model:
    T   = T_prl + max(L * (max{T_l0, T_ca1} + max{T_l1 + T_ga0, T_ca0}), T_swap) + T_pol
    T_l = interp(linear table, tokens of the sub-batch)          T_l = T_po + T_pr
    T_ga0 = interp(GPU decode table, KV tokens of batch-0's GPU decode requests)
            + sum over prefills of (a t^2 + b t)
    T_ca = interp(CPU decode table, KV tokens of the sub-batch's CPU requests)
    interp: piecewise linear, linear extrapolation, clamped >= 0, 0 for 0 tokens
Objective: throughput x / T, larger is better (the paper's "T/x" is read as
x/T, DESIGN s1).  Balancing inequalities: T_l0 >= T_ca1 and
T_l1 + T_ga0 >= T_ca0.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

WAITING, GPU_DECODE, CPU_DECODE = 0, 1, 2


@dataclass
class Profile:
    L: int
    t_prl: float
    t_pol: float
    lin: list                # [(tokens, seconds/layer)] sorted
    gdec: list               # [(kv tokens, seconds/layer)] sorted
    gpre_a: float
    gpre_b: float
    cdec: list               # [(kv tokens, seconds/layer)] sorted
    page_size: int
    max_batch_tokens: int
    pcie_bytes_per_s: float
    kv_bytes_per_token_layer: float


@dataclass
class Req:
    id: int
    kind: int                # WAITING / GPU_DECODE / CPU_DECODE
    ctx: int                 # KV tokens held (decode) or prompt tokens (waiting)


@dataclass
class Plan:
    two_batch: bool = False
    batch0: list = field(default_factory=list)
    batch1: list = field(default_factory=list)
    swap_out: list = field(default_factory=list)
    swap_in: list = field(default_factory=list)
    x: int = 0
    t_iter: float = 0.0
    t_l0: float = 0.0
    t_l1: float = 0.0
    t_ga0: float = 0.0
    t_ca0: float = 0.0
    t_ca1: float = 0.0


def interp(table, key):
    """P:279 "linear interpolation"; linear extrapolation beyond the ends,
    clamped at 0; 0 for an empty sub-batch (key 0)."""
    if key <= 0:
        return 0.0
    xs = [p[0] for p in table]
    ys = [p[1] for p in table]
    if key <= xs[0]:
        i = 0
    elif key >= xs[-1]:
        i = len(xs) - 2
    else:
        i = max(k for k in range(len(xs) - 1) if xs[k] <= key)
    x0, x1, y0, y1 = xs[i], xs[i + 1], ys[i], ys[i + 1]
    return max(0.0, y0 + (y1 - y0) * (key - x0) / (x1 - x0))


def pages(n, P):
    return (n + P - 1) // P


def iteration_time(p: Profile, t_l0, t_l1, t_ga0, t_ca0, t_ca1, t_swap):
    """P:273-275 T_tr = L (max{T_l0, T_ca1} + max{T_l1 + T_ga0, T_ca0}); plus the
    pre/post-layer constants and the swap time that layer-wise overlap cannot hide
    (DESIGN s7)."""
    t_tr = p.L * (max(t_l0, t_ca1) + max(t_l1 + t_ga0, t_ca0))
    return p.t_prl + max(t_tr, t_swap) + p.t_pol


class _State:
    """Sub-batch bookkeeping with the cost terms of P:273-279."""

    def __init__(self, p):
        self.p = p
        self.gpu_dec, self.prefill, self.cpu0, self.cpu1 = [], [], [], []

    def tokens0(self):
        return len(self.gpu_dec) + sum(r.ctx for r in self.prefill) + len(self.cpu0)

    def t_l0(self, extra=0):
        return interp(self.p.lin, self.tokens0() + extra)

    def t_l1(self, extra=0):
        return interp(self.p.lin, len(self.cpu1) + extra)

    def t_ga0(self):
        p = self.p
        pre = 0.0                       # plain left-to-right float sum (Python's sum() is compensated)
        for r in self.prefill:
            pre += p.gpre_a * r.ctx * r.ctx + p.gpre_b * r.ctx
        return interp(p.gdec, sum(r.ctx + 1 for r in self.gpu_dec)) + pre

    def t_ca0(self, extra=0):
        return interp(self.p.cdec, sum(r.ctx + 1 for r in self.cpu0) + extra)

    def t_ca1(self, extra=0):
        return interp(self.p.cdec, sum(r.ctx + 1 for r in self.cpu1) + extra)

    def balanced(self):
        """T_l0 >= T_ca1 and T_l1 + T_ga0 >= T_ca0."""
        return self.t_ca1() <= self.t_l0() and self.t_ca0() <= self.t_l1() + self.t_ga0()


def schedule(p: Profile, reqs, gpu_free: int, cpu_free: int) -> Plan:
    return _schedule(p, reqs, gpu_free, cpu_free)[0]


def state_after_step3(p: Profile, reqs, gpu_free: int, cpu_free: int):
    """(GPU decoding requests of batch-0, prefills of batch-0, CPU decoding queue)
    as step 4 sees them -- the starting point of the exhaustive bound."""
    return _schedule(p, reqs, gpu_free, cpu_free)[1]


def _schedule(p: Profile, reqs, gpu_free: int, cpu_free: int):
    P = p.page_size
    st = _State(p)
    plan = Plan()
    waiting = [r for r in reqs if r.kind == WAITING]
    gdec = [r for r in reqs if r.kind == GPU_DECODE]
    cdec = [r for r in reqs if r.kind == CPU_DECODE]
    swap_pages = 0

    # Step 1: two empty batch schedules (st: batch-0 = gpu_dec + prefill +
    # cpu0, batch-1 = cpu1).
    # Step 2: every GPU decoding request into batch-0; swap out (LIFO,
    # DESIGN s2) until the GPU can hold the new KV, or swap in (FIFO) while space
    # is ample (projected free pages stay > 0, DESIGN s3).
    grow = lambda r: pages(r.ctx + 1, P) - pages(r.ctx, P)
    need = sum(grow(r) for r in gdec)
    while need > gpu_free and gdec:
        v = gdec[-1]
        if cpu_free < pages(v.ctx, P):
            gdec.pop()                                   # cannot move it: sits out this iteration
            need -= grow(v)
            continue
        gdec.pop()
        need -= grow(v)
        gpu_free += pages(v.ctx, P)
        cpu_free -= pages(v.ctx, P)
        swap_pages += pages(v.ctx, P)
        plan.swap_out.append(v.id)
        cdec.append(Req(v.id, CPU_DECODE, v.ctx))         # now a CPU-request
    gpu_free -= need
    if not plan.swap_out:
        moved = []
        for r in cdec:
            if gpu_free - pages(r.ctx + 1, P) > 0:
                gpu_free -= pages(r.ctx + 1, P)
                cpu_free += pages(r.ctx, P)
                swap_pages += pages(r.ctx, P)
                plan.swap_in.append(r.id)
                moved.append(r)
                gdec.append(Req(r.id, GPU_DECODE, r.ctx))
            else:
                break
        cdec = [r for r in cdec if r not in moved]
    st.gpu_dec = list(gdec)

    # Step 3: pop the prefilling waitqueue into batch-0 until the batch's
    # activations (token budget) no longer fit; KV stays on the GPU if it fits,
    # else is marked for swap-out.
    marked = set()
    for w in waiting:
        if st.tokens0() + w.ctx > p.max_batch_tokens:
            break
        need_p = pages(w.ctx, P)
        if gpu_free >= need_p:
            gpu_free -= need_p
        elif cpu_free >= need_p:
            cpu_free -= need_p
            marked.add(w.id)
        else:
            break
        st.prefill.append(w)

    snapshot = (list(st.gpu_dec), list(st.prefill), list(cdec))

    # Step 4: scan the CPU decoding runqueue; each request goes to batch-1
    # (preferred, DESIGN s4) or batch-0 if the inequalities keep holding, else it
    # is skipped for this iteration.
    for r in cdec:
        if cpu_free < grow(r):
            continue
        st.cpu1.append(r)
        if st.balanced():
            cpu_free -= grow(r)
            continue
        st.cpu1.pop()
        st.cpu0.append(r)
        if st.balanced():
            cpu_free -= grow(r)
            continue
        st.cpu0.pop()

    # Step 5: remove prefilling requests whose KV would be swapped out,
    # as long as the inequalities still hold.
    for w in reversed(list(st.prefill)):
        if w.id not in marked:
            continue
        idx = st.prefill.index(w)
        st.prefill.pop(idx)
        if st.balanced():
            cpu_free += pages(w.ctx, P)
            marked.discard(w.id)
        else:
            st.prefill.insert(idx, w)
    swap_pages += sum(pages(w.ctx, P) for w in st.prefill if w.id in marked)
    plan.swap_out += [w.id for w in st.prefill if w.id in marked]
    t_swap = swap_pages * P * p.kv_bytes_per_token_layer * p.L / p.pcie_bytes_per_s

    # Step 6: the GPU-only schedule is batch-0 without the CPU decoding
    # requests of step 4; keep the schedule with the higher estimated throughput.
    t_l0, t_l1, t_ga0, t_ca0, t_ca1 = st.t_l0(), st.t_l1(), st.t_ga0(), st.t_ca0(), st.t_ca1()
    x2 = len(st.gpu_dec) + len(st.prefill) + len(st.cpu0) + len(st.cpu1)
    T2 = iteration_time(p, t_l0, t_l1, t_ga0, t_ca0, t_ca1, t_swap)
    cpu0, cpu1 = st.cpu0, st.cpu1
    st.cpu0, st.cpu1 = [], []
    t_l0_g = st.t_l0()
    x1 = len(st.gpu_dec) + len(st.prefill)
    T1 = iteration_time(p, t_l0_g, 0.0, t_ga0, 0.0, 0.0, t_swap)
    two = bool(cpu0 or cpu1) and x2 / T2 > (x1 / T1 if x1 else 0.0)
    plan.two_batch = two
    plan.batch0 = [r.id for r in st.gpu_dec] + [r.id for r in st.prefill] + ([r.id for r in cpu0] if two else [])
    plan.batch1 = [r.id for r in cpu1] if two else []
    plan.x = x2 if two else x1
    plan.t_iter = T2 if two else T1
    plan.t_l0, plan.t_l1, plan.t_ga0 = (t_l0, t_l1, t_ga0) if two else (t_l0_g, 0.0, t_ga0)
    plan.t_ca0, plan.t_ca1 = (t_ca0, t_ca1) if two else (0.0, 0.0)
    return plan, snapshot


def best_cpu_assignment(p: Profile, gpu_dec, prefill, cpu, t_swap=0.0):
    """Exhaustive search (SPEC scheduler oracle idea): every assignment of the CPU
    decoding requests to batch-0 / batch-1 / skip that satisfies the balancing
    inequalities; returns the best x / T (an upper bound for the greedy step 4)."""
    best = 0.0
    for assign in itertools.product((0, 1, 2), repeat=len(cpu)):
        st = _State(p)
        st.gpu_dec, st.prefill = list(gpu_dec), list(prefill)
        st.cpu0 = [r for r, a in zip(cpu, assign) if a == 0]
        st.cpu1 = [r for r, a in zip(cpu, assign) if a == 1]
        if not st.balanced():
            continue
        x = len(gpu_dec) + len(prefill) + len(st.cpu0) + len(st.cpu1)
        T = iteration_time(p, st.t_l0(), st.t_l1(), st.t_ga0(), st.t_ca0(), st.t_ca1(), t_swap)
        if x and x / T > best:
            best = x / T
    return best
