"""Summarise gpurun_out/dom_<wl>.ncu-rep (tools/ncu_dominant.sh) into
profiles/ncu_<wl>.json: the dominant kernel's DRAM traffic per launch next to
its algorithmic bytes (E_p x b_e), which bench.py reports as
roofline.traffic."""
import csv
import io
import json
import re
import subprocess
import sys

B_E = {"c1": 12, "c2": 12, "c3": 8, "c4": 16, "c5": 12}
KEYS = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write", "lts__t_sector_hit_rate.pct": "l2_hit_pct",
        "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
        "lts__t_requests_srcunit_tex.avg.pct_of_peak_sustained_elapsed": "lts_tex_req_pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
        "launch__registers_per_thread": "registers", "smsp__inst_executed.sum": "warp_instructions"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}

for wl in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/dom_{wl}.ncu-rep", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    m = {}
    for k, name in KEYS.items():
        if k in h:
            i = h.index(k)
            x = float(v[i].replace(",", ""))
            m[name] = x * SCALE.get(units[i], 1.0)
    txt = open(f"gpurun_out/ncu_case_{wl}.txt").read()
    ep = int(re.search(r"approximate E=\s*(\d+)", txt).group(1))
    algo = ep * B_E[wl]
    dram = int(m["dram_read"] + m["dram_write"])
    out = {
        "round": 1, "workload": wl,
        "source": f"ncu --set full --clock-control none (tools/ncu_dominant.sh {wl}): first approximate "
                  f"gather of a gg run, {ep} sparsified edges",
        "dominant_kernel": v[h.index("Kernel Name")][:90],
        "dominant_kernel_dram_bytes_per_launch": dram,
        "dominant_kernel_algo_bytes_per_launch": algo,
        "dominant_kernel_duration_ms_ncu": round(m["duration"], 4),
        "dominant_kernel_l2_hit_pct": round(m.get("l2_hit_pct", 0), 2),
        "dominant_kernel_l1_hit_pct": round(m.get("l1_hit_pct", 0), 2),
        "dominant_kernel_lts_tex_requests_pct_of_peak": round(m.get("lts_tex_req_pct", 0), 1),
        "dominant_kernel_l1tex_throughput_pct_of_peak": round(m.get("l1tex_pct", 0), 1),
        "dominant_kernel_warps_active_pct": round(m.get("warps_active_pct", 0), 1),
        "dominant_kernel_registers": int(m.get("registers", 0)),
        "dominant_kernel_warp_instructions": int(m.get("warp_instructions", 0)),
    }
    prev = {}
    try:
        prev = json.load(open(f"profiles/ncu_{wl}.json"))
    except Exception:
        pass
    for k in ("superstep_fold_stash_kernel", "check_fold_kernel_full_list", "vertex_kernel_dram_bytes_per_launch",
              "vertex_kernel_algo_bytes_per_launch"):
        if k in prev:
            out[k] = prev[k]
    json.dump(out, open(f"profiles/ncu_{wl}.json", "w"), indent=1)
    print(wl, out["dominant_kernel"], dram / algo, out["dominant_kernel_duration_ms_ncu"])
