"""Summarise `ncu --set full` captures (exported `--page raw --csv`) into profiles/.

python tools/ncu_summary.py gpurun_out/ncu profiles/ncu_full_r01.json profiles/ncu_full_r01.md

For each <name>.raw.csv: duration, DRAM bytes read+write (the roofline `traffic`), FP64
pipe utilisation, achieved occupancy, registers, spills and the top warp stall reasons.
The JSON is keyed by bench config (cfgN) for the config's dominant kernel.
"""
import csv
import io
import json
import os
import sys

KEYS = {
    "duration_ns": ["gpu__time_duration.sum"],
    "dram_read": ["dram__bytes_read.sum"],
    "dram_write": ["dram__bytes_write.sum"],
    "dram_pct_peak": ["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
    "sm_throughput_pct": ["sm__throughput.avg.pct_of_peak_sustained_elapsed"],
    "fp64_pipe_pct": ["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                      "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"],
    "dmma_pipe_pct": ["sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                      "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"],
    "dfma_inst": ["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"],
    "dadd_inst": ["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"],
    "dmul_inst": ["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"],
    "achieved_occupancy_pct": ["sm__warps_active.avg.pct_of_peak_sustained_active"],
    "registers": ["launch__registers_per_thread"],
    "grid": ["launch__grid_size"],
    "block": ["launch__block_size"],
    "smem_per_block": ["launch__shared_mem_per_block_dynamic"],
    "local_load_sectors": ["l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"],
    "local_store_sectors": ["l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum"],
    "issue_active_pct": ["sm__inst_issued.avg.pct_of_peak_sustained_active"],
    "ipc": ["sm__inst_executed.avg.per_cycle_active"],
}
STALL_PREFIX = "smsp__average_warp_latency_issue_stalled_"
STALL_PREFIX2 = "smsp__pcsamp_warps_issue_stalled_"

# capture -> bench config whose dominant kernel it is (later entries win)
CONFIG_OF = {"cfg1_svd_reg": "cfg1", "cfg2_qr_reg": "cfg2", "cfg3_svd_reg": "cfg3", "cfg4_svd_reg": "cfg4",
             "cfg5_qr_reg": "cfg5", "cfg3_svd_rr": "cfg3", "cfg2_qr_reg2": "cfg2", "cfg4d_dqr_reg": "cfg4d",
             "cfg4_svd_rr_inner": "cfg4", "cfg4d_bj_dqr_reg": "cfg4d", "cfg5_svd_rr_v": "cfg5"}


# configs whose hot path is several kernels per step: the captured launches are summed
CONFIG_SUM = {"cfg3": ["cfg3_svd_rr", "cfg3_svd_rr_v"],  # sweep kernel + V replay (svd_rr_vcol_kernel)
              "cfg4": ["cfg4_bj_gram_tma", "cfg4_svd_rr_inner", "cfg4_bj_rot_tma"],
              "cfg4d": ["cfg4d_bj_dqr_reg", "cfg4d_bj_dapply_wy", "cfg4d_bj_rot_tma"]}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def parse(path):
    text = open(path).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(text[start:]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name", "")}
    for k, names in KEYS.items():
        for nm in names:
            if nm in d and num(d[nm]) is not None:
                v = num(d[nm])
                unit = u.get(nm, "")
                if unit == "Kbyte":
                    v *= 1e3
                elif unit == "Mbyte":
                    v *= 1e6
                elif unit == "Gbyte":
                    v *= 1e9
                elif unit in ("usecond", "us"):
                    v *= 1e3
                elif unit in ("msecond", "ms"):
                    v *= 1e6
                elif unit in ("second", "s"):
                    v *= 1e9
                out[k] = v
                break
    stalls = {}
    for nm, v in d.items():
        if nm.startswith(STALL_PREFIX2) and "not_issued" not in nm and "." not in nm:
            x = num(v)
            if x:
                stalls[nm[len(STALL_PREFIX2):]] = x
    tot = sum(stalls.values()) or 1.0
    out["stall_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    return out


def main(src, js, md):
    res = {}
    for f in sorted(os.listdir(src)):
        if f.endswith(".raw.csv"):
            try:
                res[f[:-8]] = parse(os.path.join(src, f))
            except StopIteration:
                pass
    by_cfg = {}
    for name, r in sorted(res.items(), key=lambda kv: list(CONFIG_OF).index(kv[0]) if kv[0] in CONFIG_OF else -1):
        cfg = CONFIG_OF.get(name)
        if cfg:
            by_cfg[cfg] = {"kernel": r["kernel"],
                           "dram_bytes_per_launch": (r.get("dram_read", 0) + r.get("dram_write", 0)) or None,
                           "duration_ns_ncu": r.get("duration_ns"),
                           "source": f"ncu --set full capture {name} ({os.path.basename(md)})"}
    # configs whose step launches several kernels: traffic = sum over the captured launches
    for cfg, parts in CONFIG_SUM.items():
        if all(p in res for p in parts):
            by_cfg[cfg] = {"kernel": " + ".join(res[p]["kernel"].split("(")[0] for p in parts),
                           "dram_bytes_per_launch": sum(res[p].get("dram_read", 0) + res[p].get("dram_write", 0)
                                                        for p in parts),
                           "duration_ns_ncu": sum(res[p].get("duration_ns", 0) for p in parts),
                           "source": "ncu --set full captures " + ", ".join(parts) + f" ({os.path.basename(md)}); "
                                     "block configs: one launch of each kernel of a round-robin step"}
    json.dump({"captures": res, **by_cfg}, open(js, "w"), indent=1)
    lines = ["| capture | kernel | ncu dur (us) | DRAM R+W (MB) | DRAM % | FP64 pipe % | DMMA pipe % | occupancy % | regs | local ld/st sectors | top stalls |",
             "|---|---|---:|---:|---:|---:|---:|---:|---:|---|---|"]
    for name, r in res.items():
        k = r["kernel"].split("(")[0][:60]
        dram = (r.get("dram_read", 0) + r.get("dram_write", 0)) / 1e6
        st = ", ".join(f"{a} {b:.0%}" for a, b in list(r["stall_top"].items())[:4])
        lines.append(f"| {name} | `{k}` | {r.get('duration_ns', 0) / 1e3:.1f} | {dram:.2f} | {r.get('dram_pct_peak', 0):.1f} | "
                     f"{r.get('fp64_pipe_pct', float('nan')):.1f} | {r.get('dmma_pipe_pct', 0):.1f} | "
                     f"{r.get('achieved_occupancy_pct', 0):.1f} | "
                     f"{r.get('registers', 0):.0f} | {r.get('local_load_sectors', 0):.0f}/{r.get('local_store_sectors', 0):.0f} | {st} |")
    open(md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
