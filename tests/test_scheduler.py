"""NEXT-4: NEO's load-aware scheduler (neo_schedule).  The plain-Python
oracle (oracle/scheduler.py, the paper's six steps) is pinned by SPEC's worked
cost-model examples, the paper's principles and an exhaustive-search bound; the
native scheduler must then return the oracle's plan exactly."""
import math

import numpy as np
import pytest

from oracle import scheduler as osched
from paper_2411_01142_b200 import neo


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2411_01142_b200 import build
    build.build()


# ---- pins from SPEC's cost_model examples
def test_interp_spec_examples():
    t = [(1000, 0.010), (2000, 0.018)]
    assert math.isclose(osched.interp(t, 1500), 0.014)
    assert osched.interp(t, 1000) == 0.010
    assert math.isclose(osched.interp(t, 3000), 0.026)           # slope 8e-6 s/token extrapolated
    assert osched.interp(t, 0) == 0.0
    assert math.isclose(osched.interp([(64, 0.002), (256, 0.004)], 128), 0.002 + 0.002 * 64 / 192)


def _profile(**kw):
    p = dict(L=2, t_prl=0.0, t_pol=0.0, lin=[(1, 1e-4), (10000, 1.0)], gdec=[(1, 1e-9), (1e6, 1e-3)],
             gpre_a=0.0, gpre_b=1e-7, cdec=[(1, 1e-6), (1e6, 1.0)], page_size=16, max_batch_tokens=8192,
             pcie_bytes_per_s=50e9, kv_bytes_per_token_layer=4096)
    p.update(kw)
    return p


def _oprofile(d):
    return osched.Profile(d["L"], d["t_prl"], d["t_pol"], d["lin"], d["gdec"], d["gpre_a"], d["gpre_b"], d["cdec"],
                          d["page_size"], d["max_batch_tokens"], d["pcie_bytes_per_s"], d["kv_bytes_per_token_layer"])


def test_iteration_time_spec_examples():
    p = _oprofile(_profile(L=32))
    assert math.isclose(osched.iteration_time(p, 2e-3, 2e-4, 5e-4, 6e-4, 1.5e-3, 0.0), 32 * (2e-3 + 7e-4))
    p0 = _oprofile(_profile(L=1, t_prl=1e-4, t_pol=2e-4))
    assert math.isclose(osched.iteration_time(p0, 0, 0, 0, 0, 0, 0), 3e-4)
    p10 = _oprofile(_profile(L=10))
    assert math.isclose(osched.iteration_time(p10, 1e-3, 0, 1e-3, 0, 0, 0), 0.02)


def random_instance(rng):
    P = int(rng.choice([16, 32]))
    n_w, n_g, n_c = (int(x) for x in rng.integers(0, 7, size=3))
    reqs, rid = [], 0
    for kind, cnt in ((osched.GPU_DECODE, n_g), (osched.WAITING, n_w), (osched.CPU_DECODE, n_c)):
        for _ in range(cnt):
            reqs.append(osched.Req(rid, kind, int(rng.integers(1, 3000))))
            rid += 1
    order = rng.permutation(len(reqs))
    reqs = [reqs[i] for i in order]
    prof = _profile(L=int(rng.integers(1, 80)), t_prl=float(rng.uniform(0, 1e-3)),
                    lin=[(1, float(rng.uniform(1e-5, 1e-4))), (2048, float(rng.uniform(1e-3, 5e-3))),
                         (8192, float(rng.uniform(6e-3, 2e-2)))],
                    gdec=[(1, 1e-6), (1_000_000, float(rng.uniform(1e-4, 1e-2)))],
                    gpre_a=float(rng.uniform(0, 1e-9)), gpre_b=float(rng.uniform(0, 1e-7)),
                    cdec=[(1, 1e-6), (100_000, float(rng.uniform(1e-3, 5e-2)))], page_size=P,
                    max_batch_tokens=int(rng.integers(500, 10000)))
    gpu_free = int(rng.integers(0, 600))
    cpu_free = int(rng.integers(0, 2000))
    return prof, reqs, gpu_free, cpu_free


def test_oracle_principles_random():
    """Balancing / Hiding CPU hold for every two-batch plan; Greedy:
    the chosen plan's x/T >= the GPU-only plan's; the greedy step 4 never beats
    exhaustive search over (batch-0, batch-1, skip) assignments."""
    rng = np.random.default_rng(0)
    n_two = 0
    for _ in range(600):
        prof, reqs, gf, cf = random_instance(rng)
        p = _oprofile(prof)
        plan = osched.schedule(p, reqs, gf, cf)
        if plan.two_batch:
            n_two += 1
            assert plan.t_ca1 <= plan.t_l0 + 1e-18 and plan.t_ca0 <= plan.t_l1 + plan.t_ga0 + 1e-18
            # CPU time fully hidden (cost_model invariant 3): with both inequalities
            # holding, T is the pure GPU sum, or the swap time where PCIe is longer
            ctx = {r.id: r.ctx for r in reqs}
            swap_pages = sum(osched.pages(ctx[i], p.page_size) for i in plan.swap_out + plan.swap_in)
            t_swap = swap_pages * p.page_size * p.kv_bytes_per_token_layer * p.L / p.pcie_bytes_per_s
            t_layers = p.L * (plan.t_l0 + plan.t_l1 + plan.t_ga0)
            assert math.isclose(plan.t_iter, p.t_prl + max(t_layers, t_swap) + p.t_pol, rel_tol=1e-12)
            if t_swap <= t_layers:
                assert math.isclose(plan.t_iter, p.t_prl + t_layers + p.t_pol, rel_tol=1e-12)
        ids = {r.id for r in reqs}
        assert set(plan.batch0) <= ids and set(plan.batch1) <= ids
        assert not set(plan.batch0) & set(plan.batch1)
        assert plan.x == len(plan.batch0) + len(plan.batch1)
    assert n_two > 20


def test_greedy_vs_exhaustive_bound():
    """Step 4 is greedy: from the same post-step-3 state, no assignment of the CPU
    requests to (batch-0, batch-1, skip) found by exhaustive search beats the
    plan's x/T by more than the greedy loss -- and the greedy never beats the
    optimum (which would mean a violated constraint or a mis-costed plan)."""
    rng = np.random.default_rng(1)
    checked = eq = 0
    for _ in range(300):
        prof, reqs, _, _ = random_instance(rng)
        reqs = [r for r in reqs if r.kind != osched.WAITING]
        n_cpu = sum(r.kind == osched.CPU_DECODE for r in reqs)
        if n_cpu == 0 or n_cpu > 6:
            continue
        p = _oprofile(prof)
        P = p.page_size
        gf = sum(osched.pages(r.ctx + 1, P) - osched.pages(r.ctx, P) for r in reqs if r.kind == osched.GPU_DECODE)
        plan = osched.schedule(p, reqs, gf, 10**6)      # growth fits exactly: no swap-out, no swap-in
        assert not plan.swap_out and not plan.swap_in
        gpu_dec, pre, cpu = osched.state_after_step3(p, reqs, gf, 10**6)
        best = osched.best_cpu_assignment(p, gpu_dec, pre, cpu)
        got = plan.x / plan.t_iter if plan.x else 0.0
        assert got <= best * (1 + 1e-12)
        eq += got >= best * (1 - 1e-12)
        checked += 1
    assert checked > 60 and eq > checked // 2


def test_no_cpu_requests_is_gpu_only():
    p = _oprofile(_profile())
    reqs = [osched.Req(0, osched.GPU_DECODE, 100), osched.Req(1, osched.WAITING, 50)]
    plan = osched.schedule(p, reqs, 100, 100)
    assert not plan.two_batch and plan.batch0 == [0, 1] and plan.batch1 == []


def test_swap_out_lifo_when_gpu_full():
    p = _oprofile(_profile(page_size=16))
    reqs = [osched.Req(0, osched.GPU_DECODE, 32), osched.Req(1, osched.GPU_DECODE, 48)]   # both grow a page
    plan = osched.schedule(p, reqs, 1, 100)
    assert plan.swap_out == [1]                               # newest GPU-request offloads first


@pytest.mark.parametrize("seed", range(4))
def test_native_matches_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(800):
        prof, reqs, gf, cf = random_instance(rng)
        ref = osched.schedule(_oprofile(prof), reqs, gf, cf)
        got = neo.schedule(prof, [(r.id, r.kind, r.ctx) for r in reqs], gf, cf)
        assert got["two_batch"] == ref.two_batch
        assert got["batch0"] == ref.batch0 and got["batch1"] == ref.batch1
        assert got["swap_out"] == ref.swap_out and got["swap_in"] == ref.swap_in
        assert got["x"] == ref.x
        for k in ("t_iter", "t_l0", "t_l1", "t_ga0", "t_ca0", "t_ca1"):
            assert got[k] == getattr(ref, k), k


def test_native_validation():
    with pytest.raises(neo.NeoError):
        neo.schedule(_profile(lin=[(1, 0.1)]), [], 0, 0)               # < 2 points
    with pytest.raises(neo.NeoError):
        neo.schedule(_profile(lin=[(5, 0.1), (1, 0.2)]), [], 0, 0)     # decreasing keys
    with pytest.raises(neo.NeoError):
        neo.schedule(_profile(), [(0, 7, 10)], 0, 0)                    # bad kind
    assert neo.schedule(_profile(), [], 0, 0)["x"] == 0
