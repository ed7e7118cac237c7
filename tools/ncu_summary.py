"""Summarise an ncu report (--set full) into profiles/: per-kernel duration,
DRAM traffic, tensor-pipe utilisation and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/prof_r1.ncu-rep profiles/ncu_r1_summary
writes <out>.json and <out>.txt.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "utc_bf16_ops_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "tmem_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block_dynamic",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "sm_busy_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_bytes": "lts__t_bytes.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "l2_sectors_pct": "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "l2_red_input_pct": "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm_to_xbar_req_active_pct": "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm_to_xbar_write_pct": "l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed",
    "smem_lsu_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smem_tc_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12, "ms": 1, "us": 1e-3,
         "ns": 1e-6, "s": 1e3}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    result = []
    for r in rows[2:]:
        k = {"kernel": r[col["Kernel Name"]].split("(")[0]}
        for name, metric in KEYS.items():
            if metric in col:
                v = r[col[metric]].replace(",", "")
                try:
                    x = float(v)
                    u = units[col[metric]]
                    if name.endswith("bytes") or name == "l2_bytes":
                        x *= SCALE.get(u, 1)
                    if name == "duration_ms":
                        x *= SCALE.get(u, 1)
                    k[name] = x
                except ValueError:
                    k[name] = v
        stalls = {}
        for h, i in col.items():
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               (h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct")):
                try:
                    stalls[h.replace("smsp__warp_issue_stalled_", "").replace("_per_warp_active.pct", "")] = float(r[i])
                except ValueError:
                    pass
        k["top_stalls_pct"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        result.append(k)
    with open(out + ".json", "w") as f:
        json.dump(result, f, indent=1)
    with open(out + ".txt", "w") as f:
        for k in result:
            f.write(json.dumps(k) + "\n")
    for k in result:
        print(json.dumps(k))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
