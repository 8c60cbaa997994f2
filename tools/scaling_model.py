"""Schedule model of the P-rank parareal solve (contiguous slice blocks, boundary hops rank g -> g+1),
driven by per-slice phase times MEASURED on one B200 (bench.py / tools/bench_configs.py phase
breakdown).  It replays the dependency structure of driver.cu: Step 0 is a chain over all slices (each
rank continues from the boundary it receives); rank g's fine sweep k starts once its last Step-0 /
correction slice is done and runs its active slices at the per-slice fine time; correction sweep k on
rank g starts when its fine sweep ended and the upstream boundary arrived, then walks its slices.
A MODEL, not a measurement: multi-GPU scaling could not be measured (one B200 per box).

    python tools/scaling_model.py            # cfg[3] and cfg[4] at P = 1, 2, 4, 8
"""
import json


def solve_time(N, P, k_done, t_fine, t_coarse_step0, t_corr, t_hop):
    """Per-slice times in ms: fine propagation, Step-0 coarse step, correction step; t_hop: one
    boundary transfer.  Returns the modelled time-to-tol (ms)."""
    base, rem = divmod(N, P)
    blocks, s0 = [], 0
    for g in range(P):
        c = base + (1 if g < rem else 0)
        blocks.append((s0, s0 + c))
        s0 += c
    # Step 0: a chain over all slices
    ready = [0.0] * P        # time rank g's coarse stream is done with the current coarse phase
    t = 0.0
    for g, (a, b) in enumerate(blocks):
        if g > 0:
            t += t_hop
        t += (b - a) * t_coarse_step0
        ready[g] = t
    for k in range(k_done):
        fine_end = []
        for g, (a, b) in enumerate(blocks):
            active = max(0, b - max(a, k))
            fine_end.append(ready[g] + active * t_fine)
        t_up = 0.0
        for g, (a, b) in enumerate(blocks):
            active = max(0, b - max(a, k))
            if active == 0:
                continue
            start = max(fine_end[g], t_up + (t_hop if g > 0 and k < a else 0.0))
            ready[g] = start + active * t_corr
            t_up = ready[g]
    return max(ready)


def main():
    # measured per-slice phase times (ms) on one B200, round 2
    cases = {
        # cfg[4]: sqrt flow, n = 4096, N = 64, k_done = 1 (bench.py phases: ms_fine 32641 over 64 slices,
        # ms_coarse 507.6 over 64 slices, ms_correct 615.2 over 64 slices)
        "cfg4_sqrt_n4096": dict(N=64, k_done=1, t_fine=32641.0 / 64, t_coarse_step0=507.6 / 64,
                                t_corr=615.2 / 64),
        # cfg[3]: inverse flow, n = 4096, N = 64, k_done = 5 (sequential fine 254.6 s over 64 slices;
        # coarse and correction steps are one Euler step = 2 GEMMs of 3.9 ms each)
        "cfg3_inverse_n4096": dict(N=64, k_done=5, t_fine=254564.0 / 64, t_coarse_step0=7.9, t_corr=8.5),
    }
    t_hop = 0.4   # 128 MiB over NVLink 5 with 8 NCCL CTAs: an ASSUMPTION (~0.3 TB/s), not measured here
    for name, c in cases.items():
        t1 = solve_time(P=1, t_hop=t_hop, **c)
        for P in (1, 2, 4, 8):
            tp = solve_time(P=P, t_hop=t_hop, **c)
            print(json.dumps({"workload": name, "P": P, "model_time_to_tol_ms": tp,
                              "model_efficiency": t1 / (P * tp), "assumed_hop_ms": t_hop}))


if __name__ == "__main__":
    main()
