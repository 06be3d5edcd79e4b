"""Summarise scripts/ncu_variants.sh output: one row per (variant, size, kernel)
from the LAST launch of each kernel name (warm), with achieved fp32 FMA
throughput against the SIMT peak, tensor-pipe use and DRAM GB/s."""
import csv
import glob
import json
import os
import sys

PEAK_FP32 = 148 * 128 * 2 * 1.965e9 / 1e12   # TF at sm_max_mhz (MEASURED_PEAKS)


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return {}
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    last = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        key = (name, int(r[ii]))
        last.setdefault(name, {})
        last[name].setdefault(key[1], {})[r[mi]] = (r[vi].replace(",", ""), r[ui])
    return {n: d[max(d)] for n, d in last.items()}


def num(m, k, scale=None):
    if k not in m:
        return None
    v, u = m[k]
    try:
        v = float(v)
    except ValueError:
        return None
    if scale:
        v *= scale.get(u, 1.0)
    return v


def main(d):
    out = []
    for f in sorted(glob.glob(os.path.join(d, "*.csv"))):
        variant, size = os.path.basename(f)[:-4].rsplit("-", 1)
        for kern, m in load(f).items():
            if kern.startswith(("normal_kernel", "k_fill", "elementwise", "vectorized_elementwise")):
                continue
            t = num(m, "gpu__time_duration.sum", {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
                                                   "msecond": 1e-3, "nsecond": 1e-9})
            ffma = num(m, "sm__sass_thread_inst_executed_op_ffma_pred_on.sum") or 0.0
            rd = num(m, "dram__bytes_read.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}) or 0.0
            wr = num(m, "dram__bytes_write.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}) or 0.0
            row = {"variant": variant, "n": int(size), "kernel": kern, "us": round(t * 1e6, 2) if t else None,
                   "fma_pipe_pct": num(m, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                   "tf32_tensor_pct": num(m, "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off."
                                             "avg.pct_of_peak_sustained_elapsed"),
                   "sm_ghz": num(m, "sm__cycles_elapsed.avg.per_second", {"Ghz": 1, "hz": 1e-9, "Mhz": 1e-3}),
                   "dram_GBps": round((rd + wr) / t / 1e9, 1) if t else None,
                   "l2_hit_pct": num(m, "lts__t_sector_hit_rate.pct")}
            n = int(size)
            if kern.startswith(("k0", "k1", "k2", "k34", "k56", "k6", "k7")) and t:
                alg = 2.0 * n ** 3 / t / 1e12
                row["alg_TFLOPs"] = round(alg, 2)
                if kern.startswith("k7"):
                    # the kernel's own tensor-pipe utilisation at its clock: the
                    # 272.5 TF MEASURED_PEAKS-derived ceiling is exceeded by short
                    # launches (cuBLAS bf16 burst ~69 % of the 8192 flop/clk/SM rate)
                    row["bound"] = "tf32 tensor pipe (UTCHMMA ops % of peak at the kernel's clock)"
                    row["frac"] = round((row["tf32_tensor_pct"] or 0) / 100, 3)
                    row["frac_vs_measured_peaks"] = round(alg / 272.47, 3)
                else:
                    row["bound"] = f"fp32 FFMA {PEAK_FP32:.1f} TF"
                    row["frac"] = round(alg / PEAK_FP32, 3)
                if ffma:   # scalar FFMA kernels: the counter agrees with the algorithmic count
                    row["ffma_counter_TFLOPs"] = round(2 * ffma / t / 1e12, 2)
            elif t:
                row["bound"] = "HBM 6540.8 GB/s (MEASURED_PEAKS)"
                row["frac"] = round(row["dram_GBps"] / 6540.8, 3)
            out.append(row)
    return out


if __name__ == "__main__":
    for r in main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_variants"):
        print(json.dumps(r))
