"""Per-CTA timeline of the fused replay+scan kernel (globaltimer stamps), cold inputs."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import inputs  # noqa: E402
from paper_2505_14969_b200 import api, binding  # noqa: E402

binding.stree_set_launch_flags(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
prob = inputs.config_problem("c4")
layers = [api.upload(inputs.make_problem(prob.dims, prob.parent, seed=inputs.BASE_SEED + 50 + i)) for i in range(8)]
tok, vt = inputs.make_accept_inputs(prob.parent, seed=5, p_match=0.9)
path, plen, _ = api.accept(torch.from_numpy(tok).cuda(), layers[0]["parent"], torch.from_numpy(vt).cuda())
if os.environ.get("NOREPLAY"):   # path_len = 0: replay disabled (state unchanged, no state store)
    plen.zero_()
ys = [torch.empty_like(l["x"]) for l in layers]
L = binding.lib()
L.stree_debug_tc_trace.argtypes = [ctypes.c_void_p]
buf = torch.zeros((1024, 256), dtype=torch.int64, device="cuda")


def run(l, y):
    api.replay_scan(l, path, plen, l, l["h0"], y=y)


for _ in range(3):
    for l, y in zip(layers, ys):
        run(l, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    for l, y in zip(layers, ys):
        run(l, y)
e1.record()
torch.cuda.synchronize()
print(f"eager back-to-back over 8 layers: {e0.elapsed_time(e1) / 40 * 1e3:.2f} us per replay_scan")
for l, y in zip(layers[:-1], ys):
    run(l, y)
if os.environ.get("ISOLATED"):   # flush L2 and drain before the traced launch
    junk = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    if os.environ.get("ISOLATED") == "clean":   # read-only sweep: L2 ends up clean
        for _ in range(3):
            float(junk.sum())
    torch.cuda.synchronize()
buf[:, 127] = int(os.environ.get("DBG", "0"))   # kernel debug knobs (1: skip Y0 MMAs, 2: skip Y' MMAs)
L.stree_debug_tc_trace(ctypes.c_void_p(buf.data_ptr()))
run(layers[-1], ys[-1])
torch.cuda.synchronize()
L.stree_debug_tc_trace(None)
tr = buf.cpu().numpy().astype(np.int64)
n = int((tr[:, 0] > 0).sum())
tr = tr[:n]
t0 = tr[:, 0].min()
rel = np.where(tr > 0, tr - t0, -1) / 1000.0
names = {0: "start", 1: "epi start", 2: "C landed", 3: "G ready", 46: "ctf32", 50: "coefs done", 51: "BAR_G"}
for k in range(9):
    names[4 + 2 * k] = f"acc{k}"
    names[5 + 2 * k] = f"out{k}"
    names[30 + k] = f"mma_full{k}"
    names[64 + 3 * k] = f"upd_full{k}"
    names[65 + 3 * k] = f"upd_done{k}"
    names[66 + 3 * k] = f"upd_store{k}"
for k in range(9):
    names[100 + k] = f"mma_y0issued{k}"
    names[109 + k] = f"mma_x+m_ready{k}"
    names[118 + k] = f"mma_accempty{k}"
    names[91 + k] = f"built_m{k}"
for k in range(16):
    names[128 + k] = f"state_issue{k}"
for k in range(6):
    names[52 + 2 * k] = f"epi_bar{k}"
    names[53 + 2 * k] = f"epi_comp{k}"
    names[160 + k] = f"epi_tmem{k}"
names[170] = "epi_dry_start"
for k in range(9):
    names[180 + k] = f"y0_done{k}"
    names[190 + k] = f"yp_done{k}"
names[171] = "epi_dry_end"
for c in sorted(names):
    v = rel[:, c]
    v = v[v >= 0]
    if len(v):
        print(f"{names[c]:>12s}: min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
# per-CTA state-slot cycle: latency = landed (updater sees it) - issued; hold = released (next issue into
# the slot) - landed
lat, hold = [], []
for row in tr:
    for k in range(4, 9):
        iss, land = row[128 + k], row[64 + 3 * k]
        land_prev = row[64 + 3 * (k - 4)]
        if iss > 0 and land > 0:
            lat.append((land - iss) / 1000.0)
        if iss > 0 and land_prev > 0:
            hold.append((iss - land_prev) / 1000.0)
if lat:
    print(f"state load latency (issue->landed, k>=4): med {np.median(lat):.2f} us  p90 {np.percentile(lat, 90):.2f}")
    print(f"state slot hold (landed->reissued):       med {np.median(hold):.2f} us  p90 {np.percentile(hold, 90):.2f}")
