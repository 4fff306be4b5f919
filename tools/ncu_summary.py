"""Summarise an ncu report (raw page) into the metrics we track."""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sass__inst_executed_local_loads", "sass__inst_executed_local_stores", "lts__t_bytes.sum",
    "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tensor_op_dmma.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "sass__inst_executed_register_spilling",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_hit.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_miss.sum",
]
STALLS = "smsp__average_warp_latency_issue_stalled_"


def summary(rep):
    """rep: an .ncu-rep file, or the csv of `ncu -i rep --page raw --csv`."""
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, out = rows[0], rows[1], []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:90]}
        for h, u, v in zip(hdr, units, vals):
            if h in WANT or (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")):
                try:
                    d[h] = float(v.replace(",", ""))
                except ValueError:
                    d[h] = v
                if u:
                    d[h + ".unit"] = u
        out.append(d)
    return out


if __name__ == "__main__":
    res = summary(sys.argv[1])
    for d in res:
        st = {k: v for k, v in d.items() if k.startswith("smsp__pcsamp") and not k.endswith(".unit")}
        tot = sum(st.values()) or 1
        for k in [k for k in d if k.startswith("smsp__pcsamp")]:
            d.pop(k)
        d["stall_share"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(v / tot, 3)
                            for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]}
    print(json.dumps(res, indent=1))
