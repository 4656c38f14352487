"""Summaries of ncu captures for profiles/ (run here, on the .csv/.ncu-rep brought back
from the GPU box).

  python tools/summarize_ncu.py launches <launches.csv> <out.csv>
  python tools/summarize_ncu.py kernel <prof.ncu-rep> <out.txt> [traffic_json]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", ""))
        u = r[iu]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    with open(dst, "w") as f:
        f.write("kernel,launches,total_us,avg_us,share_pct\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k},{n},{t:.1f},{t / n:.1f},{100 * t / tot:.2f}\n")
    print(open(dst).read())


KEYS = ["gpu__time_duration.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum"]


def kernel(rep, dst, traffic_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    traffic = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"== {d['Kernel Name']}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k} = {d[k]} {u.get(k, '')}")
        stalls = sorted(((float(d[h]), h.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", "")) for h in hdr
            if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio") and d[h]),
            reverse=True)[:8]
        out.append("  top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1)
        wr = float(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1)
        traffic.append(rd + wr)
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))
    if traffic_json:
        json.dump({"source": rep, "bytes_per_launch_mean": sum(traffic) / len(traffic),
                   "launches": len(traffic)}, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kernel(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
