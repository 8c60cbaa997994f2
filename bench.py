"""bench.py -- parareal matrix-function solve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl mine|reference]

Workload (BASELINE.json configs[4], the n = 4096 time-to-tol config that fits one GPU in a
few-minute run): steady-state square-root flow F(X) = A - X^2, X0 = I, A = 2D 5-point Laplacian
on a 64 x 64 grid + I (n = 4096, dense FP64), T = 20, N = 64 slices, fine RK4 h = 5/512 (m_F = 32),
coarse 2 Euler steps/slice, until ||A - X^2||_F/||A||_F <= 1e-10 (checked for k >= 1, reading R10).
A "step" is one complete parareal solve (Step 0 coarse sweep, fine sweep(s), correction sweep(s),
stop metric): the whole hot path of SURVEY §8(a).  --config 3 selects the n = 4096 inverse flow
(much longer: ~20 min per solve on one GPU).

value = algorithmic fine-propagator flops of the solve (8 n^3 per RK4 step x m_F x slice-solves,
all ranks) / device time of the solve (max over ranks): FP64 TFLOP/s, whole job.  The solve's
time-to-tol is ms_per_step.  Inputs are resident in HBM (each matrix 128 MiB; the working set of
~40 GiB is far larger than L2, so no L2 flush is needed).  e2e = the same metric through the C ABI
with host buffers: mfode_set_matrix (H2D of A) + mfode_parareal_solve + mfode_get_result (D2H of X).
roofline = the dominant kernel (the fused RK-stage DMMA GEMM on the fine stream), timed by the
library with CUDA events around every fine chunk on the stream the kernels run on.
cpu_baseline = the CPU oracle (oracle/dense.py) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-propagator FP64 TFLOP/s and parareal time-to-tol at n=4096, 1/2/4/8 GPUs"
UNIT = "TFLOP/s"


INT8_PEAK_TOPS = 4553.2   # measured dense kind::i8 tcgen05 rate on this pool's B200 (tools/umma_peak.cu)


def fp64_peak():
    """FP64 tensor (DMMA) peak: MEASURED_PEAKS.json has no FP64 entry, so it is the measured chip
    peak of the mma.sync.m8n8k4.f64 register-loop probe (tools/fp64_peaks.cu), committed in
    profiles/fp64_peaks_r01.json; cuBLAS DGEMM at n = 4096 is recorded beside it."""
    p = os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")
    peak, cublas = 37.0, None
    try:
        d = json.load(open(p))
        vals = [x["tflops"] for x in d["probes"] if x.get("probe") == "dmma_m8n8k4"]
        peak = max(vals)
        cublas = [x for x in d["dgemm"] if x["n"] == 4096][0]["tflops_burst"]
    except Exception:
        pass
    return peak, cublas


def ncu_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


class ClockSampler:
    def __init__(self, device=0):
        self.samples = []
        self.proc = None
        self.device = device

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            out = ""
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            try:
                self.samples.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
            except (ValueError, IndexError):
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        loaded = sorted(s[0] for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i, v in enumerate(s[3]) if v.lower() == "active"})
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": max(s[1] for s in self.samples),
                "power_w_max": max(s[2] for s in self.samples), "samples": len(self.samples), "reasons": reasons}


def oracle_sample(w, budget_s=20.0):
    """The oracle as it stands on a bounded sample of the workload: fine RK4 steps of slice 0
    (oracle.dense.rk4 with the flow's right-hand side), repeated until ~budget_s/2 of CPU work.
    Returns (tflops, seconds, steps, threads).  Runs in whatever process calls it; bench.py calls it
    through cpu_baseline_subprocess() so that no CUDA context or torch thread pool competes."""
    import numpy as np
    from oracle import dense
    rhs = dense.make_rhs(w.A, w.flow)
    X = np.eye(w.n)
    h = w.T / (w.N * w.m_F)
    flops_step = (16.0 if w.flow == 0 else 8.0) * float(w.n) ** 3
    t0 = time.perf_counter()
    steps = 0
    while True:
        X = dense.rk4(rhs, X, h, 1)
        steps += 1
        if time.perf_counter() - t0 >= budget_s * 0.5 or steps >= 64:
            break
    dt = time.perf_counter() - t0
    threads = None
    try:
        from threadpoolctl import threadpool_info
        threads = max(i.get("num_threads", 0) for i in threadpool_info()) or None
    except Exception:
        pass
    return flops_step * steps / dt / 1e12, dt, steps, threads or os.cpu_count()


def host_description():
    """nproc, the CPU model name and the BLAS / OpenMP thread settings of this host."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model,
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


_CPU_CHILD = r"""
import json, os, sys
sys.path.insert(0, sys.argv[1])
import workloads
import bench
w = workloads.config(int(sys.argv[2]), with_eig=False)
tf, dt, steps, threads = bench.oracle_sample(w, float(sys.argv[3]))
info = {}
try:
    from threadpoolctl import threadpool_info
    info = [{k: d.get(k) for k in ("internal_api", "num_threads", "version")} for d in threadpool_info()]
except Exception:
    pass
print(json.dumps({"tflops": tf, "seconds": dt, "steps": steps, "threads": threads, "pools": info}))
"""


def cpu_baseline_subprocess(config, budget_s):
    """Time the oracle sample in a fresh Python process (no torch, no CUDA context), so the repo arm's
    cpu_baseline and the --impl reference arm measure the same program the same way."""
    out = subprocess.run([sys.executable, "-c", _CPU_CHILD, ROOT, str(config), str(budget_s)],
                         capture_output=True, text=True, timeout=600)
    if out.returncode != 0:
        raise RuntimeError(f"cpu baseline child failed: {out.stderr[-500:]}")
    d = json.loads(out.stdout.strip().splitlines()[-1])
    d.update(host_description())
    return d


def cpu_baseline_line(w, d):
    return {"value": d["tflops"], "unit": UNIT, "cores": d["threads"], "kind": "oracle",
            "sample": f"{d['steps']} RK4 step(s) of slice 0 of {w.name} with oracle.dense.rk4 "
                      f"(numpy/OpenBLAS) in a fresh process, {d['seconds']:.1f} s",
            "nproc": d["nproc"], "cpu_model": d["cpu_model"], "blas_pools": d.get("pools"),
            "OMP_NUM_THREADS": d["OMP_NUM_THREADS"], "OPENBLAS_NUM_THREADS": d["OPENBLAS_NUM_THREADS"]}


def plumbing_test(args):
    """The multi-rank harness of the bench without a GPU (tests/test_multirank_cpu.py): gloo process
    group, barrier, each rank times a token amount of host work, the max over ranks is reduced to rank 0,
    which prints one JSON line with n_gpus = WORLD_SIZE and the per-rank slice blocks."""
    import torch
    import torch.distributed as dist
    import paper_1505_07959_b200 as mf
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    ms = (time.perf_counter() - t0) * 1e3
    t = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"plumbing_test": True, "n_gpus": world, "max_rank_ms": float(t.item()),
                          "rank_slice_blocks": [list(mf.partition(64, world, r)) for r in range(world)]}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(args):
    """--gpus N without a torchrun environment: re-launch this script as N ranks (one per GPU,
    torch.distributed.run on 127.0.0.1).  Fails loudly when the box has fewer than N GPUs."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not args.plumbing_test:
        print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible", file=sys.stderr)
        return 3
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sym-steps", type=int, default=1, help="timed solves of the f3 symmetric variant (0: skip)")
    ap.add_argument("--emu-steps", type=int, default=1,
                    help="timed solves of the f3(ii) int8-tensor-core emulated variant (0: skip)")
    ap.add_argument("--emu-moduli", type=int, default=16)
    ap.add_argument("--no-seqfine", action="store_true", help="skip timing mfode_sequential_fine (the K = N reference)")
    ap.add_argument("--no-cfg2", action="store_true", help="secondary lines: skip the ~70 s cfg[2] solve")
    ap.add_argument("--no-secondary", dest="secondary", action="store_false",
                    help="skip the cfg[0] / cfg[1] iteration-dynamics lines reported beside the headline")
    ap.add_argument("--plumbing-test", action="store_true",
                    help="CPU check of the multi-rank plumbing (spawn, gloo barrier, max over ranks); no solve")
    args = ap.parse_args()

    in_torchrun = "WORLD_SIZE" in os.environ
    if not in_torchrun and args.gpus > 1 and args.impl == "mine":
        return spawn_ranks(args)
    if args.plumbing_test:
        return plumbing_test(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "mine" and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 3

    import numpy as np
    import workloads
    w = workloads.config(args.config, with_eig=False)

    if args.impl == "reference":
        # The reference arm is the CPU oracle (no reference implementation exists); rank 0 only.
        if rank != 0:
            return 0
        vals, secs = [], []
        for i in range(args.warmup + args.steps):
            d = cpu_baseline_subprocess(args.config, min(20.0, 120.0 / max(1, args.warmup + args.steps)))
            if i >= args.warmup:
                vals.append(d["tflops"])
                secs.append(d["seconds"])
        v = float(np.mean(vals))
        cpu = cpu_baseline_line(w, d)
        cpu["value"] = v
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(secs)) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "n": w.n, "N_slices": w.N, "m_G": w.m_G, "m_F": w.m_F,
                       "parallelism": "cpu"},
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return 0

    # the CPU oracle sample first, in a fresh process, before this process creates a CUDA context
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_line(w, cpu_baseline_subprocess(args.config, 20.0))
        except Exception as e:   # noqa: BLE001
            cpu = {"error": str(e)}

    import torch
    import torch.distributed as dist
    import paper_1505_07959_b200 as mf

    torch.cuda.set_device(local_rank)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        obj = [bytes(torch.cuda.nccl.unique_id()) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    solver = mf.Solver(w.A, w.flow, w.T, w.N, w.m_G, w.m_F, world=world, rank=rank, device=local_rank,
                       nccl_uid=uid)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solver.solve(w.K_max, w.tol, w.stop)
    barrier()
    infos = []
    with ClockSampler(local_rank) as clk:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record()
        for _ in range(args.steps):
            infos.append(solver.solve(w.K_max, w.tol, w.stop))
        ev1.record()
        ev1.synchronize()
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    fine_flops = float(np.mean([i["fine_flops"] for i in infos]))   # all ranks' slices (whole job)
    value = fine_flops / (ms_step * 1e-3) / 1e12

    # dominant kernel: fused RK-stage DMMA GEMM (library-timed on its own stream, this rank)
    kms = sum(i["fine_kernel_ms"] for i in infos)
    kfl = sum(i["fine_kernel_flops"] for i in infos)
    kla = sum(i["fine_kernel_launches"] for i in infos)
    achieved = kfl / (kms * 1e-3) / 1e12 if kms > 0 else None
    peak, cublas = fp64_peak()
    traffic = ncu_traffic()
    if not w.name.startswith("cfg4"):
        traffic = None   # the ncu capture is of the headline launch (13 slices of n = 4096) only

    # e2e through the C ABI with host buffers (H2D of A and D2H of X inside the timed region)
    X_host = np.empty((w.n, w.n), dtype=np.float64)
    A_host = np.ascontiguousarray(w.A)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    e2e_flops = 0.0
    for _ in range(args.e2e_steps):
        solver.set_matrix(A_host)
        inf = solver.solve(w.K_max, w.tol, w.stop)
        solver.result(X_host)
        e2e_flops += inf["fine_flops"]
    e1.record()
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = e2e_flops / (e2e_ms * 1e-3) / 1e12 if args.e2e_steps > 0 else None
    resid = solver.residual()

    def variant(opts, steps):
        """Time `steps` solves with solver options `opts` (reported beside, never folded into, value)."""
        try:
            for k, v in opts.items():
                solver.set_option(k, v)
            solver.solve(w.K_max, w.tol, w.stop)      # warm-up
            barrier()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            vinfos = [solver.solve(w.K_max, w.tol, w.stop) for _ in range(steps)]
            s1.record()
            s1.synchronize()
            vms = s0.elapsed_time(s1) / steps
            if world > 1:
                t = torch.tensor([vms], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                vms = float(t.item())
            vres = solver.residual()
            X_v = np.empty((w.n, w.n))
            solver.result(X_v)
            for k in opts:
                solver.set_option(k, 0)
            ffl = float(np.mean([i["fine_flops"] for i in vinfos]))
            vkms = sum(i["fine_kernel_ms"] for i in vinfos)
            vkfl = sum(i["fine_kernel_flops"] for i in vinfos)
            extra = {}
            if opts.get("emulation"):
                # executed int8 tensor work of the fine phase: T moduli x 2n^3 per FP64 GEMM (sym mode:
                # only the upper-triangle tiles run, reported approximately by the algorithmic count)
                ops = vkfl * opts["emulation"]
                rate = ops / (vkms * 1e-3) / 1e12 if vkms > 0 else None
                extra = {"int8_tensor_tops_fine_phase": rate, "int8_peak_tops_measured": INT8_PEAK_TOPS,
                         "int8_frac_fine_phase": (rate / INT8_PEAK_TOPS) if rate else None,
                         "int8_peak_source": "tools/umma_peak.cu (kind::i8 M128 N256 K32 from smem, 128 cyc/MMA)",
                         "note": "fine phase = encode + int8 GEMMs + CRT decode; the int8 GEMM kernel alone is "
                                 "85% tensor-pipe active in ncu (profiles/ncu_full_r01_oz_gemm.md)"}
            return {**extra, "options": opts, "time_to_tol_ms": vms, "k_done": vinfos[-1]["k_done"], "residual": vres,
                    "algorithmic_fine_tflops": ffl / (vms * 1e-3) / 1e12,
                    "fine_phase_tflops_algorithmic": (vkfl / (vkms * 1e-3) / 1e12) if vkms > 0 else None,
                    "speedup_vs_full": ms_step / vms,
                    "rel_frob_diff_vs_dmma_result": float(np.linalg.norm(X_v - X_host) / np.linalg.norm(X_host)),
                    "gpu_launches": int(sum(i["gpu_launches"] for i in vinfos))}
        except Exception as e:   # noqa: BLE001
            return {"options": opts, "error": str(e)}

    # f3(i) symmetric variant: A = A^T, so every GEMM computes only its upper-triangle tiles and
    # mirrors them (half the executed flops).
    sym = variant({"symmetric": 1}, args.sym_steps) if args.sym_steps > 0 else None
    if sym and "time_to_tol_ms" in sym:
        tiles = max(1, -(-w.n // 128))   # 128-wide tile rows (ceil): upper triangle incl. diagonal = t(t+1)/2 of t^2
        sym["executed_fine_tflops_approx"] = sym["algorithmic_fine_tflops"] * (tiles + 1) / (2 * tiles)
    # f3(ii) every GEMM (except the residual's) emulated on the int8 tensor cores (CRT/Ozaki-II, exact
    # integer products of 55-bit-scaled operands), alone and combined with f3(i)
    emu = variant({"emulation": args.emu_moduli}, args.emu_steps) if args.emu_steps > 0 else None
    emu_sym = (variant({"emulation": args.emu_moduli, "symmetric": 1}, args.emu_steps)
               if args.emu_steps > 0 else None)

    # The headline config converges at k = 1 (one fine sweep); the other BASELINE configs exercise
    # the iteration (k_done 4, 6 and 8) on the other fine-propagator kernels (K6 at n = 32, K10 at
    # n = 256, the batched DMMA GEMM with speculative next-sweep overlap at n = 1024).  Reported
    # beside the headline, one GPU (rank 0 alone), not folded into `value`.  cfg[2] is one ~64 s
    # solve (warmed by a coarse-only K = 0 solve), so it is timed once; --no-cfg2 skips it.
    secondary = None
    if world == 1 and args.secondary:
        secondary = []
        for c in ((0, 1) if args.no_cfg2 else (0, 1, 2)):
            wc = workloads.config(c, with_eig=False)
            sc = mf.Solver(wc.A, wc.flow, wc.T, wc.N, wc.m_G, wc.m_F)
            reps = 3 if c < 2 else 1
            sc.solve(wc.K_max if c < 2 else 0, wc.tol, wc.stop)   # warm-up
            ic = [sc.solve(wc.K_max, wc.tol, wc.stop) for _ in range(reps)]
            ms = float(np.mean([i["ms_total"] for i in ic]))
            sq = sc.sequential_fine()
            kf = ic[-1]
            kname = ("K6c fine_cluster_kernel (one 2-CTA cluster per slice)" if wc.n <= 64 else
                     "K10 fine_fused_kernel" if wc.n <= 512 else "dgemm_tma_kernel (batched, fused RK epilogue)")
            secondary.append({
                "workload": wc.name, "n": wc.n, "N_slices": wc.N, "k_done": kf["k_done"], "timed_solves": reps,
                "deltas": kf.get("deltas"),
                "time_to_tol_ms": ms, "fine_tflops_whole_solve": kf["fine_flops"] / (ms * 1e-3) / 1e12,
                "fine_kernel_tflops": kf["fine_kernel_flops"] / (kf["fine_kernel_ms"] * 1e-3) / 1e12,
                "fine_kernel": kname,
                "phases_ms": {k: kf.get(k) for k in ("ms_coarse", "ms_fine", "ms_correct", "ms_comm")},
                "gpu_launches_per_solve": kf["gpu_launches"], "sequential_fine_ms": sq["ms_total"],
                "speedup_vs_sequential_fine": sq["ms_total"] / ms})
            sc.close()

    # the K = N reference: sequential fine propagation through the same ranks (the
    # same work as one GPU: each rank propagates its slices in turn and hands the state on)
    seq = None
    if not args.no_seqfine:
        solver.set_option("phase_timing", 0)
        if w.n < 4096:   # small configs: one untimed call first (first-use launch set-up is ms, the solve is not)
            solver.sequential_fine()
        barrier()
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record()
        sinfo = solver.sequential_fine()
        q1.record()
        q1.synchronize()
        # the library's own device time (ev_t0..ev_t1 on the solver's streams, max over its ranks); the torch
        # events above sit on torch's current stream and only bracket the call's host time
        sq_ms = float(sinfo.get("ms_total") or q0.elapsed_time(q1))
        if world > 1:
            t = torch.tensor([sq_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sq_ms = float(t.item())
        solver.set_option("phase_timing", 1)
        seq = {"ms": sq_ms, "fine_flops": sinfo["fine_flops"],
               "tflops": sinfo["fine_flops"] / (sq_ms * 1e-3) / 1e12,
               "speedup_parareal_vs_seqfine": sq_ms / ms_step,
               "note": "T_seqfine / T_parareal(P): parareal does ~k_done x the fine work of the sequential "
                       "reference, so this is bounded by ~P / k_done (SURVEY §8(d))"}

    blocks = [list(mf.partition(w.N, world, r)) for r in range(world)]
    phases = {k: float(np.mean([i[k] for i in infos])) for k in ("ms_coarse", "ms_correct", "ms_comm", "ms_metric",
                                                                  "ms_fine", "ms_total")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "host": host_description(),
            "config": {"workload": w.name, "n": w.n, "N_slices": w.N, "m_G": w.m_G, "m_F": w.m_F, "T": w.T,
                       "stop": "residual<=1e-10 (k>=1)" if w.stop == 2 else f"stop={w.stop} tol={w.tol}",
                       "global_batch": w.N, "parallelism": f"time-slices/{world} ranks",
                       "l2": ("inputs larger than L2 (128 MiB per matrix, ~40 GiB working set); no flush"
                              if w.n >= 4096 else
                              f"parity-size config (not the headline): {8 * w.n * w.n / 2**20:.3g} MiB per matrix, "
                              "working set may sit in L2; no flush, not a bandwidth claim")},
            "time_to_tol_ms": ms_step,
            "k_done": infos[-1]["k_done"],
            "rank_slice_blocks": blocks,
            "phases_ms_rank0_mean": phases,
            "sequential_fine": seq,
            "scaling_inputs": {"T_parareal_ms": ms_step, "n_gpus": world,
                               "note": "E(P) = T_parareal(1) / (P T_parareal(P)) is computed by the driver from "
                                       "the per-N lines; ms_comm is this rank's stream time in NCCL transfers"},
            "residual": resid,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms / max(1, args.e2e_steps),
                    "h2d_bytes_per_step": 8 * w.n * w.n, "d2h_bytes_per_step": 8 * w.n * w.n},
            "gpu_launches": int(sum(i["gpu_launches"] for i in infos)),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": traffic.get("bytes_per_launch") if traffic else None,
                         "traffic_algorithmic_bytes_per_launch": traffic.get("algorithmic_bytes_per_launch")
                         if traffic else None,
                         "traffic_note": traffic.get("note") if traffic else None,
                         "kernel": ("dgemm_tma_kernel<128,128,2,4,4,EPI_RK> (fused RK4-stage FP64 DMMA GEMM)"
                                    if w.name.startswith("cfg4") else
                                    "this config's fine kernel as the library selects it (K6/K6c fine_smem for "
                                    "small n, K10 one-launch fused sweep for moderate n, else the DMMA GEMM; "
                                    "DESIGN.md kernels table)"),
                         "launches": kla, "kernel_ms": kms,
                         "peak_source": "measured FP64 DMMA probe (profiles/fp64_peaks_r01.json); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "cublas_dgemm_4096_tflops": cublas},
            "cpu_baseline": cpu,
            "f3_symmetric_variant": sym,
            "f3_emulated_variant": emu,
            "f3_emulated_symmetric_variant": emu_sym,
            "secondary_configs": secondary,
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
