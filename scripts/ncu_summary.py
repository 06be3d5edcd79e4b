"""Compact per-kernel summary of ncu reports (for profiles/).

    python scripts/ncu_summary.py gpurun_out/s2i/prof_k7_bench.ncu-rep [...] > profiles/r1/x.csv

Reads `ncu -i <rep> --page raw --csv` and keeps the counters the roofline
and the DESIGN discussion cite."""
import csv
import io
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for line in r[2:]:
        d = dict(zip(hdr, line))
        yield d, dict(zip(hdr, units))


def main():
    w = csv.writer(sys.stdout)
    w.writerow(["report", "kernel", "metric", "unit", "value"])
    for rep in sys.argv[1:]:
        for d, u in rows(rep):
            name = d.get("Kernel Name", "?")
            for k in KEEP:
                hit = [h for h in d if h.endswith(k)]
                for h in hit[:1]:
                    w.writerow([rep.split("/")[-1], name[:80], k, u.get(h, ""), d[h]])


if __name__ == "__main__":
    main()
