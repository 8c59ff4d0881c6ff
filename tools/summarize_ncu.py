"""Summarise the ncu captures of tools/profile_round.sh into profiles/ (run here, no GPU needed).

  profiles/<tag>_kernels_<cfg>.md   per-launch table: kernel, duration, DRAM bytes, DRAM %, tensor %, ...
  profiles/<tag>_launches_<cfg>.md  launch list of the bench command with each kernel family's share
  profiles/traffic.json             {cfg: {kernel family: dram bytes per launch}} (bench.py roofline.traffic)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("PROF_DIR", os.path.join(ROOT, "profiles"))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
cfgs = sys.argv[2:] or ["resnet18", "csrnet", "fsrcnn"]

METRICS = {
    "gpu__time_duration.sum": "dur_us",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_rt_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "Tbyte": 1e12, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}


def family(name):
    for f in ("fused_conv", "merged_gemm", "rowstream_conv", "tap_fold", "offset_add", "selective_add",
              "eop_affine_gather", "eop_affine_rows", "eop_affine_transpose", "eop_eval", "weight_dlt"):
        if f in name:
            return f
    return name.split("(")[0][-40:]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for m, k in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1) if k in ("dram_rd", "dram_wr", "l2_bytes", "dur_us") else v
        out.append(d)
    return out


traffic_path = os.path.join(PROF, "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for cfg in cfgs:
    rep = os.path.join(OUT, f"{tag}_full_{cfg}.ncu-rep")
    if os.path.exists(rep):
        rows = raw(rep)
        lines = [f"# {tag} ncu --set full, every libollie kernel of one `{cfg}` step",
                 "", "Captured with `tools/profile_round.sh` (`ncu --set full --clock-control none`, cold cache, "
                 "serialised replays). Bytes are per launch.", "",
                 "| # | kernel | dur us | DRAM rd MB | DRAM wr MB | DRAM % | tensor % | SM % | occ % | regs | grid |",
                 "|---|---|---|---|---|---|---|---|---|---|---|"]
        fam = defaultdict(list)
        for i, d in enumerate(rows):
            tb = d.get("dram_rd", 0) + d.get("dram_wr", 0)
            fam[family(d["kernel"])].append(tb)
            lines.append(f"| {i} | {family(d['kernel'])} | {d.get('dur_us', 0):.2f} | {d.get('dram_rd', 0)/1e6:.2f} | "
                         f"{d.get('dram_wr', 0)/1e6:.2f} | {d.get('dram_pct', 0):.1f} | "
                         f"{d.get('tensor_pct', d.get('tensor_rt_pct', 0)):.1f} | {d.get('sm_pct', 0):.1f} | "
                         f"{d.get('occ_pct', 0):.1f} | {int(d.get('regs', 0))} | {int(d.get('grid', 0))} |")
        open(os.path.join(PROF, f"{tag}_kernels_{cfg}.md"), "w").write("\n".join(lines) + "\n")
        traffic[cfg] = {k: sum(v) / len(v) for k, v in fam.items()}
        print(f"{cfg}: {len(rows)} launches profiled")
    lst = os.path.join(OUT, f"{tag}_launches_{cfg}.csv")
    if os.path.exists(lst):
        txt = "".join(l for l in open(lst) if not l.startswith("=="))
        rows = list(csv.reader(io.StringIO(txt)))
        h = rows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        tot = defaultdict(float)
        n = defaultdict(int)
        for r in rows[1:]:
            t = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1) * (1e-3 if r[ui] in ("nsecond", "ns") else 1)
            if r[ui] in ("nsecond", "ns"):
                t = float(r[vi].replace(",", "")) / 1e3
            tot[family(r[ki])] += t
            n[family(r[ki])] += 1
        ours = {k: v for k, v in tot.items() if k in ("fused_conv", "merged_gemm", "rowstream_conv", "tap_fold",
                                                      "offset_add", "selective_add", "eop_affine_gather",
                                                      "eop_affine_rows", "eop_affine_transpose", "eop_eval",
                                                      "weight_dlt")}
        s_all = sum(ours.values()) or 1.0
        lines = [f"# {tag} launch list of `python bench.py --config {cfg} --steps 2 --warmup 3 --no-graph` under "
                 "`ncu --metrics gpu__time_duration.sum --clock-control none`", "",
                 "Cold-cache, serialised per-launch times: compare each family's SHARE with bench.py's "
                 "`roofline.share_of_step` / `kernels`, not the absolute times.", "",
                 "| kernel family | launches | total us | share of libollie time |", "|---|---|---|---|"]
        for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {k} | {n[k]} | {v:.1f} | {v / s_all:.3f} |")
        others = {k: v for k, v in tot.items() if k not in ours}
        lines += ["", f"Other (torch / flush / cuDNN-free) kernels in the list: {sum(n[k] for k in others)} launches."]
        open(os.path.join(PROF, f"{tag}_launches_{cfg}.md"), "w").write("\n".join(lines) + "\n")
json.dump(traffic, open(traffic_path, "w"), indent=1)
print("traffic:", json.dumps(traffic))
