"""Write the judged summary of an ncu --set full capture to profiles/:
  python tools/ncu_to_json.py <rep> <out.json> [workload]
and record dram read+write bytes per launch in profiles/traffic.json."""
import csv, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__cycles_active.avg", "sm__cycles_active.max",
        "sm__cycles_elapsed.avg", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]

rep, out = sys.argv[1], sys.argv[2]
wl = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
res = {"kernel": d.get("Kernel Name", ""), "source_capture": rep.split("/")[-1]}
num = lambda k: float(d[k].replace(",", ""))  # noqa: E731
for k in KEYS:
    if k in d:
        res[k] = {"unit": u[h.index(k)], "value": num(k)}
stalls = {}
for i, name in enumerate(h):
    if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
        try:
            x = float(v[i])
        except ValueError:
            continue
        if x >= 0.05:
            stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
# derived: bytes through L2 per second against the LTS cap (~6300 B/cycle; the round-2
# microbenchmark tools/l2_bench.cu measured 12.75 TB/s = ~6500 B/cycle at 1.965 GHz)
t_s = num("gpu__time_duration.sum") * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}[u[h.index("gpu__time_duration.sum")]]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
dram = num("dram__bytes_read.sum") * scale[u[h.index("dram__bytes_read.sum")]] + \
    num("dram__bytes_write.sum") * scale[u[h.index("dram__bytes_write.sum")]]
l2b = num("lts__t_sectors.sum") * 32
clk = num("sm__cycles_elapsed.avg.per_second") * 1e9
res["derived"] = {"dram_bytes_per_launch": dram, "dram_GBps": dram / t_s / 1e9,
                  "l2_bytes_per_launch": l2b, "l2_TBps": l2b / t_s / 1e12,
                  "l2_cap_TBps_at_clock": 6300 * clk / 1e12, "l2_frac_of_cap": l2b / t_s / (6300 * clk)}
json.dump(res, open(out, "w"), indent=1)
if wl:
    tj = json.load(open("profiles/traffic.json"))
    tj[wl] = int(dram)
    json.dump(tj, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(res["derived"], indent=1))
