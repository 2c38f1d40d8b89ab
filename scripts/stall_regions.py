"""Warp-stall reasons and instruction counts of one ncu --set full capture, grouped by CUDA source
regions of the HVP kernel (line ranges of the files in csrc/), via nvdisasm -lineinfo.

usage: python scripts/stall_regions.py <report.ncu-rep> <kernel regex> <mangled-name substring>
"""
import collections
import csv
import io
import subprocess
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_lines import line_map  # noqa: E402

REASONS = ["stall_barrier", "stall_wait", "stall_short_sb", "stall_long_sb", "stall_math", "stall_selected",
           "stall_not_selected", "stall_mio", "stall_dispatch", "stall_branch_resolving", "stall_lg", "stall_no_inst"]


def region(fn, ln, src_lines):
    if fn is None:
        return "?"
    text = src_lines.get(fn, {}).get(ln, "")
    if fn == "tiled.cuh" and TILED_ITEM[0] <= ln <= TILED_ITEM[1]:
        return "phase2 item (weights load + FMA)"
    if fn == "hvp_sw.cuh":
        for lo, hi, name in REGIONS_SW:
            if lo <= ln <= hi:
                return name
    if fn == "tiled.cuh" and 225 <= ln <= 237:
        return "phase1 store weights"
    if fn in ("tiled.cuh", "device.cuh") and ("bspline" in text or "base_of" in text or ln in range(80, 101)):
        return "phase1 weights"
    return f"{fn}:{ln}"


REGIONS_SW = []
TILED_ITEM = [0, 0]


def main():
    rep, kre, fsub = sys.argv[1:4]
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    csrc = os.path.join(root, "paper_2605_09097_b200", "csrc")
    src = {}
    for f in os.listdir(csrc):
        src[f] = {i + 1: t for i, t in enumerate(open(os.path.join(csrc, f)).read().splitlines())}
    # phase-2 item helpers of tiled.cuh: from `struct ItemW` to `item_quadratic`
    tl = src["tiled.cuh"]
    TILED_ITEM[0] = next(i for i, t in tl.items() if "struct ItemW" in t)
    TILED_ITEM[1] = next(i for i, t in tl.items() if "item_quadratic(" in t)
    # regions of hvp_sw.cuh by marker comments / function names
    lines = src["hvp_sw.cuh"]

    def find(s):
        for i, t in lines.items():
            if s in t:
                return i
        return None
    g0 = find("void sw_gather")
    e0 = find("void sw_emit")
    f0 = find("void sw_flush") or find("struct FlushItem")  # the flush became FlushItem::flush
    k0 = find("k_hvp_sw(")
    c0 = find("// M2 = A gd^T")
    c1 = find("__syncthreads();  // records ready")
    p2 = next(i for i, t in sorted(lines.items()) if i > c1 and "if (it < T::ITEMS) {" in t)
    em = find("node plane `layer` is complete")
    pf0 = find("void sw_prefetch")
    REGIONS_SW.extend([(pf0, pf0 + 18, "TMA issue (sw_prefetch)"), (g0, e0 - 1, "phase1 gather"), (e0, f0 - 1, "emit"), (f0, f0 + 60, "flush"),
                       (find("void sw_prefetch_tmap"), find("void sw_prefetch_tmap") + 20, "TMA issue (tensor map)"),
                       (c0, c1 - 1, "phase1 constitutive+store G"), (c1, p2 - 1, "records barrier + TMA issue"),
                       (p2, em - 1, "phase2 loop control"), (em, em + 10, "emit/flush barriers"),
                       (k0, c0 - 1, "tile setup + phase1 loads")])
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hi = his[0]
    end = his[1] - 1 if len(his) > 1 else len(rows)
    h = rows[hi]
    data = [r for r in rows[hi + 1:end] if len(r) == len(h)]
    amap = line_map(fsub)
    a0 = int(data[0][0], 16)
    idx = {k: h.index(k) for k in REASONS if k in h}
    iE = h.index("Instructions Executed")
    agg = collections.defaultdict(lambda: collections.Counter())

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    for r in data:
        key = amap.get(int(r[0], 16) - a0, (None, 0))
        reg = region(key[0], key[1], src)
        for k, i in idx.items():
            agg[reg][k] += f(r[i])
        agg[reg]["inst"] += f(r[iE])
    tot_st = sum(sum(v for k, v in c.items() if k != "inst") for c in agg.values()) or 1
    tot_in = sum(c["inst"] for c in agg.values()) or 1
    print(f"{'region':40s} {'stall%':>6s} {'inst%':>6s}  " + " ".join(k.replace("stall_", "")[:8].rjust(8) for k in idx))
    for reg, c in sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "inst")):
        st = sum(v for k, v in c.items() if k != "inst")
        if st / tot_st < 0.005 and c["inst"] / tot_in < 0.005:
            continue
        print(f"{reg[:40]:40s} {st / tot_st * 100:6.1f} {c['inst'] / tot_in * 100:6.1f}  " +
              " ".join(f"{c[k] / tot_st * 100:8.1f}" for k in idx))


if __name__ == "__main__":
    main()
