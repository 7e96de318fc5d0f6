"""Summarise an ncu capture and a launch list into profiles/ (run here, no GPU needed).

    python tools/ncu_summarize.py --rep gpurun_out/prof_c4.ncu-rep --launches gpurun_out/launches.csv \
        --tag r01_c4 [--json profiles/ncu_summary.json]
"""
from __future__ import annotations

import argparse
import csv
import io
import re
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_bytes.sum",
           "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "nsecond": 1e-9}


def kernel_key(name: str, order: str = "A") -> str:
    if "gemm1_mpo_fused" in name:
        return "gemm1_mpo_fused_A"
    if "gemm_cluster_splitk" in name:
        return "gemm_cluster_splitk"
    if "mpo_apply_kernel" in name:
        return f"mpo_{order}"
    if "gemm_dmma_tma_kernel" in name and order == "B":
        kmajor = re.search(r"gemm_dmma_tma_kernel<[^>]*,\s*(\d)\s*>", name)
        return "gemm_first_B" if (kmajor and kmajor.group(1) == "1") else "gemm_last_B"
    if "gemm_dmma_tma_kernel" in name:
        # template args <BM, BN, WM, WN, STAGES, B_KMAJOR>: order A's first GEMM is NN, its last is NT
        kmajor = re.search(r"gemm_dmma_tma_kernel<[^>]*,\s*(\d)\s*>", name)
        return "gemm_last_A" if (kmajor and kmajor.group(1) == "1") else "gemm_first_A"
    if "mpo_orderA" in name:
        return "mpo_A"
    if "mpo_orderB" in name:
        return "mpo_B"
    return name.split("(")[0].split()[-1]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = None
                u = units[i]
                if v is not None and u in SCALE:
                    v = v * SCALE[u]
                    u = "s" if u in ("ns", "us", "usecond", "ms", "msecond", "nsecond", "second") else ("B" if "byte" in u else u)
                d[m] = (v, u)
        res.append(d)
    return res


def launches(path: str):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Name", "Metric Unit"))
    agg = {}
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        agg.setdefault(r[ki].split("(")[0], []).append(v)
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--json", default=str(ROOT / "profiles" / "ncu_summary.json"))
    ap.add_argument("--order", default="A", choices=["A", "B"], help="matvec order the capture ran (kernel keys)")
    ap.add_argument("--commit", default=None, help="git commit the captured build was made from")
    ap.add_argument("--build", default=None, help="libheff.so source hash of the captured build")
    args = ap.parse_args()
    md = [f"# ncu summary {args.tag}\n"]
    js = json.loads(Path(args.json).read_text()) if Path(args.json).exists() else {}
    if args.launches:
        agg = launches(args.launches)
        tot = sum(sum(v) for v in agg.values())
        md.append("## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)\n")
        md.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k}` | {len(v)} | {sum(v) * 1e3:.3f} | {sum(v) / tot:.4f} |")
        md.append("")
    if args.rep:
        md.append(f"## `ncu --set full` capture ({Path(args.rep).name})\n")
        for d in raw(args.rep):
            md.append(f"### `{d['kernel'][:110]}`\n")
            for m in METRICS:
                if m in d and d[m][0] is not None:
                    v, u = d[m]
                    md.append(f"- {m} = {v:.6g} {u}")
            rb = d.get("dram__bytes_read.sum", (None,))[0]
            wb = d.get("dram__bytes_write.sum", (None,))[0]
            if rb is not None and wb is not None and rb == rb and wb == wb:
                key = kernel_key(d["kernel"], args.order)
                js[key] = {"dram_bytes_per_launch": rb + wb, "kernel": d["kernel"][:120], "tag": args.tag,
                           "duration_s": d.get("gpu__time_duration.sum", (None,))[0],
                           "commit": args.commit, "build": args.build}
            md.append("")
    out = ROOT / "profiles" / f"{args.tag}_ncu.md"
    out.write_text("\n".join(md) + "\n")
    Path(args.json).write_text(json.dumps(js, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main()
