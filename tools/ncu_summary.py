"""Summarise an ncu --set full capture: time, DRAM bytes, hit rates, issue, stalls."""
import csv, subprocess, sys

def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "launch__registers_per_thread",
            "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "smsp__average_warp_latency_per_inst_issued.ratio"]
    for v in rows[2:]:
        d = dict(zip(h, v))
        print(d.get("Kernel Name", "")[:70])
        for k in keys:
            if k in d:
                print(f"   {k:55s} {u[h.index(k)]:10s} {d[k]}")
        st = []
        for i, name in enumerate(h):
            if "smsp__average_warps_issue_stalled" in name and name.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(v[i]), name.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("   stalls/issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:9]))

for rep in sys.argv[1:]:
    summary(rep)
