"""Summarise ncu output for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/launches_r01.md
    python tools/ncu_summary.py full gpurun_out/prof_rk.ncu-rep  > profiles/ncu_full_r01.md

`launches`: per-kernel count, total / mean device time and share of all profiled launches
(ncu per-launch times are cold-cache and serialised: compare SHARES, not absolutes).
`full`: the headline metrics of a --set full capture (duration, DRAM bytes, DMMA/tensor-pipe and
FP64 pipe utilisation, occupancy, registers, shared memory, stall reasons) per profiled launch,
plus profiles/ncu_traffic.json (bytes per launch) that bench.py reports as roofline.traffic.
"""
import csv
import collections
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    m = re.search(r"oz_gemm_kernel<(\d)>", name) or re.search(r"oz_gemm_kernelILi(\d)E", name)
    if m:
        return "oz_gemm_kernel<%s> (int8 tcgen05, %s)" % (m.group(1), "CTA pair" if m.group(1) == "1" else "1 CTA")
    m = re.search(r"dgemm_tma_kernel<(.*?)>", name)
    if m:
        return f"dgemm_tma_kernel<{m.group(1)}>"
    m = re.search(r"dgemm_tma_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)E", name)
    if m:
        epi = ["STORE", "RK", "EULER", "EULER_CORR", "RESID"][int(m.group(6))]
        return f"dgemm_tma_kernel<{m.group(1)}x{m.group(2)}, warps {m.group(3)}x{m.group(4)}, EPI_{epi}>"
    return name.split("(")[0][:90]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
        total += ns
    print(f"# ncu launch list: {os.path.basename(path)}\n")
    print(f"{sum(a[0] for a in agg.values())} profiled launches, {total / 1e6:.2f} ms total device time "
          "(cold-cache, serialised)\n")
    print("| kernel | launches | total ms | mean us | share |")
    print("|---|---|---|---|---|")
    for k, (c, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {c} | {ns / 1e6:.3f} | {ns / c / 1e3:.1f} | {100 * ns / total:.1f}% |")


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "int8 (imma) tensor pipe %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "TMEM active %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2 -> SM bytes (TMA)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("smsp__cycles_active.avg", "SMSP active cycles"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1] if len(rows) > 1 else []
    data = rows[2:]
    print(f"# ncu --set full: {os.path.basename(path)}\n")
    kname = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
    traffic = []
    for r in data:
        print(f"## {short(r[kname]) if kname is not None else '?'}\n")
        print("| metric | value | unit |")
        print("|---|---|---|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {label} (`{m}`) | {r[i]} | {units[i] if i < len(units) else ''} |")
        # stall reasons (top)
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or h.startswith("smsp__pcsamp_warps_issue_stalled_"):
                try:
                    st.append((float(r[i].replace(",", "")), h))
                except ValueError:
                    pass
        st.sort(reverse=True)
        if st:
            print("\nTop stall reasons:\n")
            for v, h in st[:8]:
                print(f"- `{h}`: {v}")
        print()
        try:
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
            ur = units[hdr.index("dram__bytes_read.sum")]
            uw = units[hdr.index("dram__bytes_write.sum")]
            traffic.append(rd * mult.get(ur, 1) + wr * mult.get(uw, 1))
        except (ValueError, IndexError):
            pass
    names = [r[kname] for r in data] if kname is not None else []
    if traffic and names and all("dgemm_tma_kernel" in nm for nm in names):   # the bench's dominant kernel only
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
            json.dump({"source": os.path.basename(path), "bytes_per_launch": sum(traffic) / len(traffic),
                       "launches": len(traffic)}, f, indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
