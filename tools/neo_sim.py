"""Iteration-level estimate of NEO's throughput gain on B200 (the paper's headline
metric) from the measured cost profile: every iteration is
planned by the native neo_schedule and its estimated time is charged; the
GPU-only baseline is the same scheduler with no CPU-cache (NEO degenerates to
vLLM-style GPU-only serving).  Offline synthetic workload per P:364: input and
output lengths uniform in [0.9 l, 1.1 l].

python tools/neo_sim.py [profile.json] [n_requests] [l_in] [l_out] [cpu_speedup]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2411_01142_b200 import neo  # noqa: E402

WAITING, GPU_DECODE, CPU_DECODE = 0, 1, 2


def pages(n, P):
    return (n + P - 1) // P


def simulate(prof, reqs, gpu_pages, cpu_pages, max_iters=200000):
    P = prof["page_size"]
    state = {i: {"in": a, "out": o, "ctx": 0, "gen": 0, "where": None} for i, (a, o) in enumerate(reqs)}
    waiting = list(range(len(reqs)))
    gpu_run, cpu_run = [], []
    gfree, cfree = gpu_pages, cpu_pages
    t = 0.0
    tokens = 0
    iters = two = 0
    while (waiting or gpu_run or cpu_run) and iters < max_iters:
        order = [(i, GPU_DECODE, state[i]["ctx"]) for i in gpu_run] + \
                [(i, WAITING, state[i]["in"]) for i in waiting] + \
                [(i, CPU_DECODE, state[i]["ctx"]) for i in cpu_run]
        plan = neo.schedule(prof, order, gfree, cfree)
        iters += 1
        two += plan["two_batch"]
        # GPU decoding requests the plan could neither grow nor move (no room in
        # either cache) are preempted by recompute, as a GPU-only engine does:
        # pages freed, back to the front of the waitqueue with the generated
        # tokens folded into the prompt.
        served = set(plan["batch0"]) | set(plan["batch1"]) | set(plan["swap_out"])
        stuck = [i for i in gpu_run if i not in served]
        for i in stuck:
            s = state[i]
            gfree += pages(s["ctx"], P)
            gpu_run.remove(i)
            s["in"], s["out"], s["ctx"], s["gen"], s["where"] = s["ctx"], s["out"] - s["gen"], 0, 0, None
            waiting.insert(0, i)
        if plan["x"] == 0:
            if stuck:
                continue
            break
        # apply swaps
        for i in plan["swap_in"]:
            s = state[i]
            cfree += pages(s["ctx"], P)
            gfree -= pages(s["ctx"], P)
            s["where"] = "gpu"
            cpu_run.remove(i)
            gpu_run.append(i)
        pre_out = set()
        for i in plan["swap_out"]:
            s = state[i]
            if s["where"] == "gpu":
                gfree += pages(s["ctx"], P)
                cfree -= pages(s["ctx"], P)
                s["where"] = "cpu"
                gpu_run.remove(i)
                cpu_run.append(i)
            else:
                pre_out.add(i)               # prefill whose KV goes to the CPU-cache
        for i in plan["batch0"] + plan["batch1"]:
            s = state[i]
            if s["where"] is None:           # prefill: KV of the prompt, first token out
                s["ctx"] = s["in"]
                if i in pre_out:
                    s["where"] = "cpu"
                    cfree -= pages(s["ctx"], P)
                    cpu_run.append(i)
                else:
                    s["where"] = "gpu"
                    gfree -= pages(s["ctx"], P)
                    gpu_run.append(i)
                waiting.remove(i)
            else:                            # decode: append one token
                grow = pages(s["ctx"] + 1, P) - pages(s["ctx"], P)
                if s["where"] == "gpu":
                    gfree -= grow
                else:
                    cfree -= grow
                s["ctx"] += 1
            s["gen"] += 1
            if s["gen"] >= s["out"]:
                if s["where"] == "gpu":
                    gfree += pages(s["ctx"], P)
                    gpu_run.remove(i)
                else:
                    cfree += pages(s["ctx"], P)
                    cpu_run.remove(i)
                s["where"] = "done"
        t += plan["t_iter"]
        tokens += plan["x"]
    done = sum(1 for s in state.values() if s["where"] == "done")
    assert done == len(reqs), f"simulation stopped with {len(reqs) - done} unfinished requests"
    return tokens / t, iters, two


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "cost_profile_b200_llama8b.json")
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    l_in = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
    l_out = int(sys.argv[4]) if len(sys.argv) > 4 else 300
    prof = json.load(open(path))
    speedup = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
    if speedup != 1.0:                   # hypothetical host: CPU attention `speedup` x faster
        prof = dict(prof, cdec=[[k, t / speedup] for k, t in prof["cdec"]])
    rng = np.random.default_rng(7)
    lo_i, hi_i = (9 * l_in + 9) // 10, (11 * l_in) // 10
    lo_o, hi_o = (9 * l_out + 9) // 10, (11 * l_out) // 10
    reqs = list(zip(rng.integers(lo_i, hi_i + 1, n).tolist(), rng.integers(lo_o, hi_o + 1, n).tolist()))
    page_bytes = prof["page_size"] * prof["kv_bytes_per_token_layer"] * prof["L"]
    cpu_pages = int(512e9 // page_bytes)
    print(f"{prof['model']} on {prof['gpu']}: {n} requests, input ~{l_in}, output ~{l_out}; "
          f"CPU-cache 512 GB ({prof.get('host_threads')} host threads, CPU attention x{speedup:g})")
    # GPU-only + swap: same scheduler and CPU-cache, CPU attention priced out of
    # reach, so CPU-resident requests only wait to be swapped back in (the
    # vLLM-with-swap-space baseline); its gap to NEO isolates CPU attention.
    noattn = dict(prof, cdec=[[1, 1e3], [2, 2e3]])
    print("| GPU KV budget | GPU-only, recompute | GPU-only + swap | NEO | NEO vs GPU+swap | two-batch iterations |")
    print("|---|---|---|---|---|---|")
    for gb in (4, 8, 16, 40, 150):
        gpages = int(gb * 1e9 // page_bytes)
        base, _, _ = simulate(prof, reqs, gpages, 0)
        swap_tp, _, _ = simulate(noattn, reqs, gpages, cpu_pages)
        neo_tp, iters, two = simulate(prof, reqs, gpages, cpu_pages)
        print(f"| {gb} GB | {base:.0f} | {swap_tp:.0f} | {neo_tp:.0f} | {100 * (neo_tp / swap_tp - 1):+.1f} % "
              f"| {two}/{iters} |")


if __name__ == "__main__":
    main()
