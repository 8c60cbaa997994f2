"""FP64 roofline measurement on one B200.

Runs the DMMA/DFMA register-loop probes (tools/fp64_peaks.cu) and times cuBLAS DGEMM through
torch.matmul(float64) as the vendor bar, sampling SM clocks during the run. Writes one JSON object
to stdout (and to the path given by --out). MEASURED_PEAKS.json is driver-owned and has no FP64
entry, so this file is where the FP64 denominator used by bench.py comes from.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import torch


def dgemm(n, reps=10, sustain_s=0.0):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out = {"n": n, "best_ms": best, "tflops_burst": 2 * n**3 / best / 1e9}
    if sustain_s > 0:
        cnt = 0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.time()
        while time.time() - t0 < sustain_s:
            for _ in range(4):
                torch.matmul(a, b, out=c)
            cnt += 4
            torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        out["tflops_sustained"] = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/fp64_peaks.json")
    ap.add_argument("--probe-bin", default="tools/fp64_peaks")
    args = ap.parse_args()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    clk = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    res = {"probes": [], "dgemm": []}
    if os.path.exists(args.probe_bin):
        p = subprocess.run([args.probe_bin], capture_output=True, text=True)
        for line in p.stdout.splitlines():
            try:
                res["probes"].append(json.loads(line))
            except json.JSONDecodeError:
                res["probes"].append({"raw": line})
        if p.returncode != 0:
            res["probe_error"] = p.stderr[-2000:]
    for n in (1024, 2048, 4096, 8192):
        res["dgemm"].append(dgemm(n, sustain_s=4.0 if n in (4096, 8192) else 0.0))
    clk.terminate()
    samples = []
    for line in clk.stdout.read().splitlines():
        parts = [x.strip() for x in line.split(",")]
        try:
            samples.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3]))
        except (ValueError, IndexError):
            pass
    if samples:
        loaded = sorted(s[0] for s in samples if s[2] > 300) or sorted(s[0] for s in samples)
        res["clocks"] = {"sm_mhz_median_loaded": loaded[len(loaded) // 2],
                         "sm_max_mhz": max(s[1] for s in samples),
                         "power_w_max": max(s[2] for s in samples),
                         "reasons": sorted({s[3] for s in samples})}
    res["gpu"] = torch.cuda.get_device_name(0)
    txt = json.dumps(res, indent=1)
    print(txt)
    with open(args.out, "w") as f:
        f.write(txt)


if __name__ == "__main__":
    sys.exit(main())
