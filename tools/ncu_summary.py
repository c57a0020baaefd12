"""Summarise an ncu --set full report into the profiles/ text format.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep "title" > profiles/rN_x_ncu_summary.txt

Prints, per captured kernel: duration, SM frequency, tensor-pipe utilisation, DRAM bytes and
throughput, L2 hit rate, achieved occupancy, registers, shared memory, grid/block and the
top stall reasons (from the raw page)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_active_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_elapsed_pct"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform_pipe_pct"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpu_dram_throughput_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster_x"),
]


def main():
    rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full --clock-control none summary: {title}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"\n## kernel: {d.get('Kernel Name', '?')[:140]}")
        for k, name in KEYS:
            if k in d:
                print(f"{name:28s} {d[k]} {u.get(k, '')}")
        stalls = [(float(d[k] or 0), k) for k in hdr
                  if k.startswith("smsp__average_warp_latency_issue_stalled_") or
                  (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"))]
        stalls = [s for s in stalls if s[0] > 0]
        for v, k in sorted(stalls, reverse=True)[:6]:
            print(f"stall {k.split('stalled_')[-1]:22s} {v}")


if __name__ == "__main__":
    main()
