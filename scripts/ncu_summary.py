"""Summarise ncu captures into profiles/ (tracked):
  python scripts/ncu_summary.py full <report.ncu-rep> <kernel-regex> <out.json>
  python scripts/ncu_summary.py launches <launches.csv> <out.json>
The `full` summary carries dram bytes per launch (bench.py's roofline.traffic), duration, pipe
utilisation, shared-memory wavefronts / bank conflicts and the warp-stall breakdown."""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second"]


def full(rep, kre, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kre}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = {"report": rep, "kernel_regex": kre, "launches": []}
    for v in rows[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        ent = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                try:
                    ent[k] = float(d[k].replace(",", ""))
                    ent[k + ".unit"] = u[k]
                except ValueError:
                    ent[k] = d[k]
        stalls = {}
        for k, val in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(val)
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        ent["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])
                            if v / tot > 0.005}
        res["launches"].append(ent)
    first = res["launches"][0]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = first["dram__bytes_read.sum"] * scale.get(first.get("dram__bytes_read.sum.unit", "byte"), 1.0)
    wr = first["dram__bytes_write.sum"] * scale.get(first.get("dram__bytes_write.sum.unit", "byte"), 1.0)
    res["dram_bytes_per_launch"] = rd + wr
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in first.items() if k != "kernel"}, indent=0)[:1500])


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ik = h.index("Kernel Name")
    iv = h.index("Metric Value")
    iu = h.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        ns = v * {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1.0)
        tot[name] += ns
        cnt[name] += 1
    s = sum(tot.values())
    res = {"source": path, "total_ms": s / 1e6, "kernels": [
        {"kernel": k, "launches": cnt[k], "ms": tot[k] / 1e6, "share": tot[k] / s} for k, _ in tot.most_common()]}
    json.dump(res, open(out, "w"), indent=1)
    for e in res["kernels"][:12]:
        print(f"{e['share'] * 100:6.2f}%  {e['ms']:9.3f} ms  x{e['launches']:5d}  {e['kernel']}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(*sys.argv[2:5])
    else:
        launches(*sys.argv[2:4])
