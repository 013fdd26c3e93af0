"""Summarise the ncu outputs of tools/profile_round.sh (run where ncu -i works)."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    per = defaultdict(lambda: defaultdict(list))
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        per[name][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    return per


API = {"lat_kernel<128, 1": "stree_replay_scan", "lat_kernel<64, 1": "stree_replay_scan",
       "lat_kernel<128, 0": "stree_tree_scan", "lat_kernel<64, 0": "stree_tree_scan",
       "lat_kernel<128, true": "stree_replay_scan", "lat_kernel<64, true": "stree_replay_scan",
       "lat_kernel<128, false": "stree_tree_scan", "lat_kernel<64, false": "stree_tree_scan",
       "scan_tc_kernel<128, 1>": "stree_replay_scan", "scan_tc_kernel<64, 1>": "stree_replay_scan",
       "scan_tc_kernel<128, 0>": "stree_tree_scan", "scan_tc_kernel<64, 0>": "stree_tree_scan",
       "scan_tc_kernel<128, 2>": "stree_commit", "scan_tc_kernel<64, 2>": "stree_commit",
       "commit_ring_kernel": "stree_commit", "commit_block_kernel": "stree_commit",
       "build_mask_kernel": "stree_build_mask", "accept_kernel": "stree_accept",
       "attn_tc_kernel": "stree_tree_attn", "attn_simt_kernel": "stree_tree_attn", "kv_commit_kernel": "stree_kv_commit",
       "tree_conv_kernel": "stree_tree_conv", "conv_commit_kernel": "stree_conv_commit", "mss_kernel": "stree_accept_mss",
       "attn_db_kernel": "stree_tree_attn"}


def api_name(k):
    for pre, v in API.items():
        pre2 = pre.rstrip(">")   # templates may carry more arguments (scan_tc_kernel<128, 1, NoYPeers>)
        if k.split("::")[-1].startswith(pre2) or pre in k or pre2 + "," in k:
            return v
    if "scan_simt" in k:
        return "stree_tree_scan"
    return k


traffic = {}
nf = os.path.join(out, "launches_nofuse.csv")
if os.path.exists(nf):
    print("== launch list, unfused order (bench.py --no-fuse) ==")
    pn = launches(nf)
    tn = sum(sum(m["gpu__time_duration.sum"]) for m in pn.values())
    for k, m in sorted(pn.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        t = m["gpu__time_duration.sum"]
        rd = sum(m["dram__bytes_read.sum"]) / len(t)
        wr = sum(m["dram__bytes_write.sum"]) / len(t)
        print(f"{k[:60]:60s} n={len(t):4d} mean={sum(t) / len(t) / 1e3:8.2f} us  share={sum(t) / tn * 100:5.1f}%  "
              f"dram r/w per launch {rd / 1e6:7.2f} / {wr / 1e6:7.2f} MB")
        traffic.setdefault(api_name(k), rd + wr)
nx = os.path.join(out, "launches_next.csv")
if os.path.exists(nx):
    print("== launch list, SURVEY §8(f) rows (tools/prof_attn.py = bench_next at 4 layers) ==")
    px = launches(nx)
    for k, m in sorted(px.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        t = m["gpu__time_duration.sum"]
        rd = sum(m["dram__bytes_read.sum"]) / len(t)
        wr = sum(m["dram__bytes_write.sum"]) / len(t)
        tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", [0.0])
        print(f"{api_name(k):18s} {k[:50]:50s} n={len(t):4d} mean={sum(t) / len(t) / 1e3:8.2f} us  "
              f"dram r/w per launch {rd / 1e6:7.2f} / {wr / 1e6:7.2f} MB  tensor pipe {sum(tp) / len(tp):5.1f}%")
        traffic.setdefault(api_name(k), rd + wr)
print("== launch list (ncu --cache-control none, serialised): per-kernel mean over launches ==")
per = launches(os.path.join(out, "launches.csv"))
tot = sum(sum(m["gpu__time_duration.sum"]) for m in per.values())
for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = m["gpu__time_duration.sum"]
    rd = sum(m["dram__bytes_read.sum"]) / len(t)
    wr = sum(m["dram__bytes_write.sum"]) / len(t)
    print(f"{k[:60]:60s} n={len(t):4d} mean={sum(t) / len(t) / 1e3:8.2f} us  share={sum(t) / tot * 100:5.1f}%  "
          f"dram r/w per launch {rd / 1e6:7.2f} / {wr / 1e6:7.2f} MB")
    traffic.setdefault(api_name(k), rd + wr)


def details(rep, names):
    try:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    except Exception as e:  # noqa: BLE001
        return str(e)
    rows = list(csv.reader(txt.splitlines()))
    if not rows:
        return "(no data)"
    hdr = rows[0]
    res = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in names:
            res.append(f"  {d.get('ID', '')} {d['Metric Name']:45s} {d['Metric Value']} {d.get('Metric Unit', '')}")
    return "\n".join(res)


names = {"Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
         "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "L2 Hit Rate", "Achieved Active Warps Per SM",
         "Issued Warp Per Scheduler", "No Eligible"}
full = {}
for rep in ("prof_fused", "prof_scan", "prof_commit", "prof_lat_c3", "prof_attn", "prof_conv"):
    p = os.path.join(out, rep + ".ncu-rep")
    if os.path.exists(p):
        print(f"== ncu --set full: {rep} ==")
        print(details(p, names))
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv", "--metrics",
                              "dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum"],
                             capture_output=True, text=True).stdout
        print(raw[-2000:])
        # per-launch DRAM bytes of the --set full capture (first captured launch)
        rows = list(csv.reader(raw.splitlines()))
        if len(rows) > 2:
            hdr = rows[0]
            d = dict(zip(hdr, rows[2]))
            try:
                unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                tot = sum(float(d[m].replace(",", "")) * unit.get(dict(zip(hdr, rows[1]))[m], 1)
                          for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                full[api_name(d.get("Kernel Name", rep))] = tot
            except (KeyError, ValueError):
                pass
# traffic = DRAM read + write per launch from the launch list (steady state, caches not flushed: the
# write-back of a launch's dirty lines lands in the following launches, so the mean is the per-launch
# traffic).  A --set full capture replays the kernel ~40 times: with flushed caches its writes stay in
# L2 (under-counted), without flushing its replays hit L2 -- kept for reference only.
print("traffic per launch (bytes, launch list):", json.dumps(traffic))
print("--set full capture DRAM bytes (replayed, reference only):", json.dumps(full))
res = {"c4": traffic, "source": "ncu launch list of bench.py, --cache-control none, mean read+write per launch"}
# batch-1 configs (small-batch kernel): launch lists of bench.py --config c3 / c2
for cfg in ("c3", "c2"):
    pf = os.path.join(out, f"launches_{cfg}.csv")
    if os.path.exists(pf):
        print(f"== launch list, bench.py --config {cfg} ==")
        pc = launches(pf)
        tc_ = sum(sum(m["gpu__time_duration.sum"]) for m in pc.values())
        tr = {}
        for k, m in sorted(pc.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
            t = m["gpu__time_duration.sum"]
            rd = sum(m["dram__bytes_read.sum"]) / len(t)
            wr = sum(m["dram__bytes_write.sum"]) / len(t)
            print(f"{k[:60]:60s} n={len(t):4d} mean={sum(t) / len(t) / 1e3:8.2f} us  share={sum(t) / tc_ * 100:5.1f}%  "
                  f"dram r/w per launch {rd / 1e6:7.2f} / {wr / 1e6:7.2f} MB")
            tr.setdefault(api_name(k), rd + wr)
        res[cfg] = tr
print("traffic.json:", json.dumps(res))
json.dump(res, open(os.path.join(out, "traffic.json"), "w"), indent=1)
