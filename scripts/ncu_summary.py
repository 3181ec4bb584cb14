"""Summarise an ncu report (.ncu-rep) and a launch-list CSV into profiles/ (run here, no GPU).
usage: python scripts/ncu_summary.py TAG [gpurun_out/prof_TAG.ncu-rep] [gpurun_out/launches_TAG.csv]"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "gpc__cycles_elapsed.max",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__t_bytes.sum",
        "smsp__inst_executed_pipe_alu.sum", "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_lsu.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            # some metrics carry a section prefix in the raw page (TPC.TriageCompute.<metric>)
            i = hdr.index(k) if k in hdr else next((j for j, h in enumerate(hdr) if h.endswith("." + k)), None)
            if i is not None:
                d[k] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


def launches(path):
    if not os.path.exists(path):
        return []
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    start = rows.index(hdr) + 1
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    return [(r[ki], float(r[vi].replace(",", ""))) for r in rows[start:] if len(r) > vi]


def main():
    tag = sys.argv[1]
    rep = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    lc = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    summ = {"tag": tag, "full_capture": raw(rep) if os.path.exists(rep) else []}
    ls = launches(lc)
    tot = sum(t for _, t in ls)
    by = {}
    for k, t in ls:
        name = k.split("(")[0]
        by.setdefault(name, [0, 0.0])
        by[name][0] += 1
        by[name][1] += t
    summ["launch_list"] = {"total_ns": tot, "kernels": {k: {"launches": n, "ns": t, "share": round(t / tot, 4) if tot else None}
                                                       for k, (n, t) in sorted(by.items(), key=lambda x: -x[1][1])}}
    out_dir = os.environ.get("NCU_OUT", os.path.join(ROOT, "profiles"))  # gpurun_out when run on the box
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"ncu_{tag}.json")
    json.dump(summ, open(out, "w"), indent=1)
    print(json.dumps(summ, indent=1)[:4000])
    if os.path.exists(rep) and os.environ.get("NCU_SOURCE"):
        # per-line source view (SASS + CUDA correlation) of the captured kernel, for stall analysis
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        open(os.path.join(out_dir, f"source_{tag}.csv"), "w").write(src)


if __name__ == "__main__":
    main()
