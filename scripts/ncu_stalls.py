"""Stall-reason shares and a few headline metrics from an ncu report."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
d = dict(zip(r[0], r[2]))
st = []
for k, x in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((float(x.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(a for a, _ in st) or 1
print("  ".join(f"{k}={100 * a / tot:.1f}%" for a, k in sorted(st, reverse=True)[:9]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__t_sector_hit_rate.pct"]:
    print(f"  {k} = {d.get(k)}")
