"""Key metrics of one-kernel `ncu --set full` reports (read here with `ncu -i ... --page raw`).

    python scripts/ncu_full_summary.py gpurun_out/r01_lm_head.ncu-rep [...] [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("duration_us", "gpu__time_duration.sum", 1e-3),
    ("sm_clock_ghz", "sm__cycles_elapsed.avg.per_second", 1.0),
    ("dram_read_bytes", "dram__bytes_read.sum", 1.0),
    ("dram_write_bytes", "dram__bytes_write.sum", 1.0),
    ("dram_throughput_pct", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("tensor_pipe_active_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("tma_l2_to_smem_bytes", "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", 1.0),
    ("l2_hit_rate_pct", "lts__t_sector_hit_rate.pct", 1.0),
    ("registers_per_thread", "launch__registers_per_thread", 1.0),
    ("threads_per_block", "launch__block_size", 1.0),
    ("grid_size", "launch__grid_size", 1.0),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "nsecond": 1, "usecond": 1e3,
        "msecond": 1e6, "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"report": path, "kernel": vals[hdr.index("Kernel Name")].split("(")[0]}
    for key, name, scale in METRICS:
        if name in hdr:
            i = hdr.index(name)
            v = float(vals[i].replace(",", ""))
            out[key] = v * UNIT.get(units[i], 1.0) * scale
    out["dram_bytes"] = out.get("dram_read_bytes", 0) + out.get("dram_write_bytes", 0)
    return out


def main():
    args = sys.argv[1:]
    jpath = None
    if "--json" in args:
        jpath = args[args.index("--json") + 1]
        args = args[: args.index("--json")]
    res = [summarize(p) for p in args]
    print("| kernel | us | SM GHz | DRAM read MB | DRAM write MB | DRAM % | tensor % | TMA L2->smem GB | L2 hit % |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in res:
        print(f"| {r['kernel']} | {r.get('duration_us', 0):.1f} | {r.get('sm_clock_ghz', 0):.2f} | "
              f"{r.get('dram_read_bytes', 0) / 1e6:.1f} | {r.get('dram_write_bytes', 0) / 1e6:.1f} | "
              f"{r.get('dram_throughput_pct', 0):.1f} | {r.get('tensor_pipe_active_pct', 0):.1f} | "
              f"{r.get('tma_l2_to_smem_bytes', 0) / 1e9:.2f} | {r.get('l2_hit_rate_pct', 0):.1f} |")
    if jpath:
        with open(jpath, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
