"""Per-source-line instruction and stall profile of one kernel from an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_MANGLED [UNIT_EXEC] [N]

Maps the SASS page of the report (--page source --print-source sass: executed instructions
and warp-stall samples per address) to kernels.cu lines through the -lineinfo tables of the
library's cubin (nvdisasm -g), and prints the N heaviest lines with the opcodes they issue.
UNIT_EXEC (e.g. the execution count of an instruction that runs once per partition) scales
the counts to "per unit".  The library must be the exact build the report was taken on.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_map(lib, kern):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "api" not in f]
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub[0])], capture_output=True,
                             text=True).stdout.splitlines()
    start = [i for i, l in enumerate(txt) if ("." + kern + " --") in l or (kern + " --") in l][0]
    cur, amap = None, {}
    for l in txt[start + 1:]:
        if l.startswith("//---------------------"):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            amap[int(m.group(1), 16)] = cur
    return amap


def main():
    rep, lib, kern = sys.argv[1:4]
    unit = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    n = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    base = int(data[0][ia], 16)
    amap = line_map(lib, kern)
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    ops = collections.defaultdict(collections.Counter)
    te = ts = 0
    for r in data:
        e, s = int(r[iex] or 0), int(r[iss] or 0)
        te += e
        ts += s
        k = amap.get(int(r[ia], 16) - base, ("?", 0))
        agg[k][0] += e
        agg[k][1] += s
        toks = r[isrc].split()
        if toks:
            ops[k][toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]] += e
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_2104_09075_b200", "csrc", "kernels.cu")).read().splitlines()
    print(f"instructions executed {te} ({te / unit:.1f} per unit), stall samples {ts}")
    for (f, ln), (e, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
        t = src[ln - 1].strip()[:64] if f == "kernels.cu" and ln > 0 else ""
        top = ", ".join(f"{o} {c / unit:.1f}" for o, c in ops[(f, ln)].most_common(3))
        print(f"{f}:{ln:<5d} {e / unit:7.1f}/unit {s / ts * 100:5.2f}% stalls | {t} | {top}")


if __name__ == "__main__":
    main()
