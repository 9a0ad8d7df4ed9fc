"""Summarise the artefacts of tools/gpu_profile_pass.sh (gpurun_out/) into profiles/ (tracked)."""
import collections
import csv
import json
import shutil
import subprocess
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"
OUT = "profiles"


def ncu(rep, page):
    return subprocess.run(["ncu", "-i", f"gpurun_out/{rep}.ncu-rep", "--page", page, "--csv"],
                          capture_output=True, text=True).stdout


raw = ncu(f"prof_scan_{TAG}", "raw")
raw_vec4 = ncu(f"prof_vec4_{TAG}", "raw")
open(f"{OUT}/{TAG}_k_scan_flowcache_raw.csv", "w").write(raw)
open(f"{OUT}/{TAG}_k_scan_flowcache_details.csv", "w").write(ncu(f"prof_scan_{TAG}", "details"))
open(f"{OUT}/{TAG}_k_scan_vec4_mode2_raw.csv", "w").write(raw_vec4)
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum',
        'l1tex__m_xbar2l1tex_read_sectors_mem_global_op_tma_ld.sum', 'lts__t_sectors.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_red.sum',
        'lts__t_sectors_srcunit_tex_op_write.sum', 'lts__t_requests_srcunit_ltcfabric.sum',
        'lts__t_requests_srcunit_tex.sum', 'lts__t_requests_srcunit_tex_op_read.sum',
        'lts__t_requests_srcunit_tex_op_red.sum', 'lts__t_requests_srcunit_tex_op_write.sum',
        'lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum', 'lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'sm__cycles_elapsed.avg', 'smsp__inst_executed.sum',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio']


def pick(text):
    rows = list(csv.reader(text.splitlines()))
    d, u = dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))
    return {k: (float(d[k].replace(',', '')) if d.get(k) not in (None, '') else None, u.get(k)) for k in KEYS}


summary = {
    "k_scan_vec4<5,2> (scan mode test_agg, no flow cache)": pick(raw_vec4),
    "k_scan_flowcache<5,SoaSource> (scan mode auto/flow_cache: 32 MiB table of 32-bit (cand, h1(opp)) keys, "
    "8 ways per sector, TMA-staged packet stream)": pick(raw),
}
json.dump(summary, open(f"{OUT}/{TAG}_scan_kernels_ncu_summary.json", "w"), indent=1)
conv = {'Mbyte': 1e6, 'Gbyte': 1e9, 'Kbyte': 1e3, 'byte': 1}


def dram(entry):
    return sum(entry[k][0] * conv[entry[k][1]] for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum'))


vec4, fc = list(summary.values())
traffic = {
    "source": f"ncu --set full captures summarised in profiles/{TAG}_scan_kernels_ncu_summary.json (one 100M-packet launch)",
    "k_scan_flowcache<5>": {"dram_bytes_per_launch": dram(fc), "algorithmic_bytes_per_launch": 8e8,
                            "note": "the 32 MiB key table and the 10 MiB sketch stay L2-resident: DRAM traffic is the packet stream"},
    "k_scan_vec4<5,2>": {"dram_bytes_per_launch": dram(vec4), "algorithmic_bytes_per_launch": 8e8},
}
json.dump(traffic, open(f"{OUT}/{TAG}_traffic.json", "w"), indent=1)
# what bench.py's roofline block reads: requests and REDs per packet of the scan kernels, from these captures
PACKETS = 100_000_000


def counters(entry, what):
    g = lambda k: entry[k][0]
    return {
        "packets_per_launch": PACKETS,
        "l2_requests_per_packet": g('lts__t_requests_srcunit_tex.sum') / PACKETS,
        "l2_read_requests_per_packet": g('lts__t_requests_srcunit_tex_op_read.sum') / PACKETS,
        "l2_red_per_packet": g('lts__t_requests_srcunit_tex_op_red.sum') / PACKETS,
        "l2_write_requests_per_packet": g('lts__t_requests_srcunit_tex_op_write.sum') / PACKETS,
        "l2_sectors_per_packet": (g('lts__t_sectors_srcunit_tex_op_read.sum') + g('lts__t_sectors_srcunit_tex_op_red.sum') +
                                  g('lts__t_sectors_srcunit_tex_op_write.sum')) / PACKETS,
        "tma_stream_sectors_per_packet": g('l1tex__m_xbar2l1tex_read_sectors_mem_global_op_tma_ld.sum') / PACKETS,
        "remote_die_requests_per_packet": g('lts__t_requests_srcunit_ltcfabric.sum') / PACKETS,
        "request_port_busy_pct": g('l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed'),
        "lts_throughput_pct": g('lts__throughput.avg.pct_of_peak_sustained_elapsed'),
        "dram_throughput_pct": g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'),
        "issue_active_pct": g('smsp__issue_active.avg.pct_of_peak_sustained_active'),
        "warp_instructions_per_packet": g('smsp__inst_executed.sum') / PACKETS,
        "gpu_time_us": g('gpu__time_duration.sum'),
        "registers_per_thread": g('launch__registers_per_thread'),
        "source": f"ncu --set full --clock-control none, one {PACKETS}-packet launch of bench.py's config-2 window ({what}); "
                  f"raw export profiles/{TAG}_{what}_raw.csv; counters lts__t_requests_srcunit_tex[_op_read|_op_red|_op_write].sum, "
                  f"l1tex__m_l1tex2xbar_req_cycles_active, lts__throughput, gpu__dram_throughput",
    }


json.dump({"k_scan_flowcache<5>": counters(fc, "k_scan_flowcache"), "k_scan_vec4<5,2>": counters(vec4, "k_scan_vec4_mode2")},
          open(f"{OUT}/{TAG}_scan_counters.json", "w"), indent=1)
for k, v in fc.items():
    print(k, v)
print("traffic", traffic)

shutil.copy(f"gpurun_out/launches_{TAG}.csv", f"{OUT}/{TAG}_launch_list_bench_steps2.csv")
for name in ("", "_reference", "_test_agg", "_test", "_red", "_config3"):
    shutil.copy(f"gpurun_out/bench_{TAG}{name}.json", f"{OUT}/{TAG}_bench{name}.json")
for src, dst in ((f"feed_probe_{TAG}.json", f"{TAG}_host_feed_probe.json"), (f"l2_probe_{TAG}.json", f"{TAG}_l2_probe.json"),
                 (f"soak_{TAG}.txt", f"{TAG}_soak.txt")):
    shutil.copy(f"gpurun_out/{src}", f"{OUT}/{dst}")
for src, dst in ((f"config3_{TAG}.json", f"{TAG}_config3_1b_packet_window.json"),
                 (f"config4_{TAG}.json", f"{TAG}_config4_ddos_contention.json"),
                 (f"config5_{TAG}.json", f"{TAG}_config5_accuracy_sweep.json"),
                 (f"tools_{TAG}.json", f"{TAG}_tools.json")):
    shutil.copy(f"gpurun_out/{src}", f"{OUT}/{dst}")
rows = [r for r in csv.reader(open(f"{OUT}/{TAG}_launch_list_bench_steps2.csv")) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].replace('dhsa::', '').replace('void ', '')
    if not name.startswith('k_'):      # this library's kernels (torch's generators and fills are not ours)
        continue
    a = agg.setdefault(name.split('(')[0][:62], [0, 0.0, []])
    a[0] += 1
    a[1] += float(r[vi].replace(',', ''))
    a[2].append(float(r[vi].replace(',', '')))
tot = sum(a[1] for a in agg.values())
lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none; python bench.py --steps 2 --warmup 3 (5 windows of 100M packets)",
         "# our kernels only (torch's data-generation kernels omitted); per-launch times are cold-cache and serialised",
         "# (the first window of a fresh sketch is a device-gated auto launch: a 2^20-packet sample through k_scan_flowcache,",
         "#  k_auto_decide, k_scan_vec4<5,1> returning at once, k_scan_flowcache over the rest -- hence 6 cache launches for 5 windows)",
         f"{'kernel':64s} {'launches':>8s} {'avg_us':>10s} {'median_us':>10s} {'share_of_our_gpu_time':>22s}"]
for k, (n, tt, each) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{k:64s} {n:8d} {tt / n / 1e3:10.2f} {sorted(each)[len(each) // 2] / 1e3:10.2f} {tt / tot:22.4f}")
open(f"{OUT}/{TAG}_launch_shares.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
