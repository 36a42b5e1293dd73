"""Summarise ncu artefacts into profiles/ (text + json).

usage: python scripts/summarize_ncu.py launches <launches.csv> <out_prefix>
       python scripts/summarize_ncu.py full <report.ncu-rep> <out_prefix> [rows_per_launch]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, data = rows[0], rows[1:]
    iname, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        v = float(r[iv].replace(",", ""))
        ns = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[iu], 1) * v
        agg[r[iname]][0] += 1
        agg[r[iname]][1] += ns
        tot += ns
    res = {"launches": len(data), "total_ms": tot / 1e6,
           "kernels": [{"name": k, "count": c, "ms": ns / 1e6, "share": ns / tot}
                       for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1])]}
    json.dump(res, open(out + ".json", "w"), indent=1)
    with open(out + ".txt", "w") as f:
        f.write(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
        f.write(f"# {len(data)} launches, {tot / 1e6:.2f} ms total\n")
        for k in res["kernels"]:
            f.write(f"{k['count']:6d} {k['ms']:10.3f} ms {100 * k['share']:6.2f}%  {k['name'][:150]}\n")
    print(open(out + ".txt").read()[:3000])


KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
]


def full(path, out, rows=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows_csv = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows_csv[0], rows_csv[1]
    res = {"report": path, "kernels": []}
    for r in rows_csv[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"name": d.get("Kernel Name"), "metrics": {}}
        for key in KEYS:
            if key in d:
                k["metrics"][key] = f"{d[key]} {u.get(key, '')}".strip()
        st = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(d[h].replace(",", "") or 0)
              for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        k["stall_share"] = {a: round(b / tot, 4) for a, b in sorted(st.items(), key=lambda kv: -kv[1])[:10]}
        if rows:
            try:
                sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
                byt = sum(float(d[key].replace(",", "")) * sc.get(u[key], 1)  # each metric has its own unit
                          for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                k["dram_bytes_per_row"] = byt / rows
            except Exception:
                pass
        res["kernels"].append(k)
    json.dump(res, open(out + ".json", "w"), indent=1)
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
