"""Attribute ncu per-SASS-instruction metrics (warp-stall samples, executed instructions) to CUDA
source lines, using nvdisasm's -lineinfo annotations of the built libosmpm.so.

usage: python scripts/sass_lines.py <report.ncu-rep> <kernel regex> <mangled-name substring> [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_09097_b200", "libosmpm.so")


def line_map(func_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
    amap = {}
    cur_fun = None
    cur_line = None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fun = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fun and func_sub in cur_fun:
            amap[int(m.group(1), 16)] = cur_line
    return amap


def main():
    rep, kre, fsub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                             f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csvtxt)))
    his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hi = his[0]
    end = his[1] - 1 if len(his) > 1 else len(rows)
    h = rows[hi]
    data = [r for r in rows[hi + 1:end] if len(r) == len(h)]
    iS = h.index("Warp Stall Sampling (All Samples)")
    iE = h.index("Instructions Executed")
    iW = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
    amap = line_map(fsub)

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    st = collections.Counter()
    ex = collections.Counter()
    wf = collections.Counter()
    a0 = int(data[0][0], 16)  # ncu reports absolute addresses; the function starts at the first
    for r in data:
        a = int(r[0], 16) - a0
        key = amap.get(a, ("?", 0))
        st[key] += f(r[iS])
        ex[key] += f(r[iE])
        if iW is not None:
            wf[key] += f(r[iW])
    ts = sum(st.values()) or 1
    te = sum(ex.values()) or 1
    tw = sum(wf.values()) or 1
    print(f"total shared wavefronts {sum(wf.values()):.4g}")
    src = {}
    order = wf if os.environ.get("SORT") == "smem" else st
    for k, _ in order.most_common(top):
        fn, ln = k
        path = os.path.join(ROOT, "paper_2605_09097_b200", "csrc", fn)
        if fn not in src and os.path.exists(path):
            src[fn] = open(path).read().splitlines()
        text = src.get(fn, [""] * (ln + 1))[ln - 1].strip()[:80] if ln else ""
        print(f"{st[k] / ts * 100:5.1f}% stall {ex[k] / te * 100:5.1f}% inst {wf[k] / tw * 100:5.1f}% smem  {fn}:{ln}  {text}")


if __name__ == "__main__":
    main()
