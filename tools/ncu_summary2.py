"""Summarise a round-2 `ncu --set full` capture of one gg run (tools/ncu_r2.sh)
into profiles/ncu_<wl>.json: per captured launch the duration, DRAM traffic
and the request-path / pipe utilisations that bound it; the first approximate
gather is the dominant kernel whose DRAM bytes per launch bench.py reports as
roofline.traffic (next to its algorithmic bytes).

    python tools/ncu_summary2.py gpurun_out/r2_c5.ncu-rep c5 gpurun_out/r2_case_c5.txt
"""
import csv
import io
import json
import re
import subprocess
import sys

B_E = {"c1": 12, "c2": 12, "c3": 8, "c4": 16, "c5": 12}
KEYS = {
    "gpu__time_duration.sum": "ms",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_requests_srcunit_tex.sum": "l2_requests",
    "lts__t_sectors_srcunit_tex.sum": "l2_sectors",
    "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed": "l2_tag_req_avg_pct",
    "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed": "l2_tag_req_max_slice_pct",
    "lts__t_tag_requests.min.pct_of_peak_sustained_elapsed": "l2_tag_req_min_slice_pct",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed": "l1_to_xbar_req_pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1_data_wavefronts_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__icc_request_hit_rate.pct": "icache_hit_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6,
         "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0, "s": 1e3}


def main(rep, wl, case_txt):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    stall_keys = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio")]
    launches = []
    for v in rows[2:]:
        m = {"kernel": v[h.index("Kernel Name")][:100]}
        for k, name in KEYS.items():
            if k in h and v[h.index(k)]:
                i = h.index(k)
                x = float(v[i].replace(",", ""))
                x *= SCALE.get(units[i], 1.0)
                m[name] = round(x, 4) if abs(x) < 1e6 else int(x)
        st = sorted(((float(v[h.index(k)]), k[len("smsp__average_warps_issue_stalled_"):-len(
            "_per_issue_active.ratio")]) for k in stall_keys if v[h.index(k)]), reverse=True)
        m["top_stalls_per_issue"] = {k: round(x, 2) for x, k in st[:5]}
        launches.append(m)
    txt = open(case_txt).read()
    ep = [int(x) for x in re.findall(r"approximate E=\s*(\d+)", txt)]
    dom = next(m for m in launches if "edge_kernel<" in m["kernel"] and ", 0>" in m["kernel"])
    algo = ep[0] * B_E[wl]
    dram = int(dom["dram_read"] + dom["dram_write"])
    out = {
        "round": 2, "workload": wl,
        "source": f"ncu --set full --clock-control none --import-source on (tools/ncu_r2.sh): the engine "
                  f"launches of one gg run (python tools/ncu_case.py --workload {wl} --iters 7), "
                  f"cold-cache serialised replays",
        "dominant_kernel": dom["kernel"],
        "dominant_kernel_dram_bytes_per_launch": dram,
        "dominant_kernel_algo_bytes_per_launch": algo,
        "dominant_kernel_edges_per_launch": ep[0],
        "dominant_kernel_duration_ms_ncu": dom["ms"],
        "dominant_kernel_l2_requests_per_edge": round(dom["l2_requests"] / ep[0], 4),
        "launches": launches,
    }
    json.dump(out, open(f"profiles/ncu_{wl}.json", "w"), indent=1)
    print(wl, dom["kernel"], "dram/algo", round(dram / algo, 3), "ms", dom["ms"])


if __name__ == "__main__":
    main(*sys.argv[1:4])
