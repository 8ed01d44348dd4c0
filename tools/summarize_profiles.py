"""Turn gpurun_out/ ncu artefacts into the committed summaries under profiles/.

    python tools/summarize_profiles.py TAG [--k5a gpurun_out/k5a_TAG.ncu-rep] [--launches ...]

Writes profiles/launches_cfg2_TAG.txt (per-kernel share of an ncu launch list),
profiles/k5a_ncu_cfg2_TAG.txt (key counters of the K5a full capture) and
profiles/k5a_traffic_CONFIG.json (dram read + write bytes of that launch, read by bench.py).
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct", "smsp__inst_executed_pipe_fp64.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmma_pred_on.sum", "smsp__inst_executed_op_shared_ld.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path, tag, note, cfg="cfg2"):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = re.sub(r"\(.*", "", re.sub(r"^void ", "", r[ki]))
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = ["# ncu launch list (gpu__time_duration.sum, --clock-control none) " + note,
           "# cold-cache serialised per-launch times; kernel  launches  total_ms  share"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append("%-64s %5d %10.3f %5.1f%%" % (k, n, v / 1e6, 100 * v / tot))
    out.append("%-64s %5s %10.3f" % ("TOTAL", "", tot / 1e6))
    dst = os.path.join(ROOT, "profiles", "launches_%s_%s.txt" % (cfg, tag))
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:12]))


def _sha():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    return bench.k5a_source_sha()


def k5a(rep, tag, note, cfg="cfg2"):
    if rep.endswith(".csv"):  # the raw page exported on the GPU box (tools/gpu_final.sh)
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {a: (b, c) for a, b, c in zip(h, u, v)}
    out = ["# ncu --set full --clock-control none --import-source on " + note, "Kernel Name  " + m["Kernel Name"][1]]
    for k in KEYS:
        if k in m:
            out.append("%-84s %s %s" % (k, m[k][1], m[k][0]))
    for k in sorted(m):
        if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                if float(m[k][1]) > 0.05:
                    out.append("%-84s %s" % (k, m[k][1]))
            except ValueError:
                pass
    open(os.path.join(ROOT, "profiles", "k5a_ncu_%s_%s.txt" % (cfg, tag)), "w").write("\n".join(out) + "\n")
    print("\n".join(out))
    rd = float(m["dram__bytes_read.sum"][1].replace(",", "")) * SCALE[m["dram__bytes_read.sum"][0]]
    wr = float(m["dram__bytes_write.sum"][1].replace(",", "")) * SCALE[m["dram__bytes_write.sum"][0]]
    json.dump({"what": "dram__bytes_read.sum + dram__bytes_write.sum of one K5a launch (%s), ncu --set full"
               % m["Kernel Name"][1].split("(")[0], "bytes_per_launch": rd + wr, "read": rd, "write": wr,
               "source": os.path.basename(rep) + " (" + tag + ")", "k5a_source_sha": _sha()},
              open(os.path.join(ROOT, "profiles", "k5a_traffic_%s.json" % cfg), "w"), indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--note", default=None)
    a = ap.parse_args()
    note = a.note or ("%s, python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --pcg-tol 0 --config %s"
                      % (a.config, a.config))
    sfx = a.tag if a.config == "cfg2" else "%s_%s" % (a.config, a.tag)
    launches(os.path.join(ROOT, "gpurun_out", "launches_%s.csv" % sfx), a.tag, note, a.config)
    rep = os.path.join(ROOT, "gpurun_out", "k5a_%s.ncu-rep" % sfx)
    if not os.path.exists(rep):
        rep = os.path.join(ROOT, "gpurun_out", "k5a_%s.raw.csv" % sfx)
    k5a(rep, a.tag, note, a.config)
