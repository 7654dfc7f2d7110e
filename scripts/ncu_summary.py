"""Key metrics of an `ncu --set full` capture, one line per profiled launch:
python scripts/ncu_summary.py rep.ncu-rep  (needs the ncu CLI)."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "us", 1e-3),
        ("dram__bytes_read.sum", "MB_rd", 1e-6),
        ("dram__bytes_write.sum", "MB_wr", 1e-6),
        ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
        # tcgen05 (UTCHMMA) bf16 tensor-op throughput: the counter that sees
        # the 5th-gen tensor cores (sm__pipe_tensor_cycles_active does not)
        ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "tc05%", 1),
        ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum", "GFLOP_tc05", 1e-9),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1),
        ("launch__grid_size", "grid", 1),
        ("launch__registers_per_thread", "regs", 1)]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    print(f"# {path}")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0].replace("delta_k::<unnamed>::", "")
        vals = []
        for k, lab, sc in KEYS:
            v = d.get(k, "")
            try:
                v = f"{float(v.replace(',', '')) * sc:.1f}"
            except ValueError:
                pass
            vals.append(f"{lab}={v}")
        print(f"{name:34s} " + " ".join(vals))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
