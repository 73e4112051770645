"""Group the SASS of one ncu report into straight-line runs of equal execution count and
print the heaviest runs (instructions executed, share, stall samples, opcode mix).

python tools/ncu_blocks.py REPORT.ncu-rep [TOP] [--show N]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 25
    show = 0
    if "--show" in sys.argv:
        show = int(sys.argv[sys.argv.index("--show") + 1])
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    ins = []
    for r in rows:
        if len(r) > 3 and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].startswith("0x"):
            d = dict(zip(hdr, r))
            ins.append((int(r[0], 16), r[1].strip(), int(d["Instructions Executed"] or 0),
                        int(d["Warp Stall Sampling (All Samples)"] or 0)))
    ins.sort()
    total = sum(i[2] for i in ins)
    samples = sum(i[3] for i in ins)
    blocks = []
    cur = []
    for x in ins:
        if cur and (x[2] != cur[-1][2]):
            blocks.append(cur)
            cur = []
        cur.append(x)
    if cur:
        blocks.append(cur)
    print(f"total warp instructions {total:.4g}, stall samples {samples}, sass lines {len(ins)}")
    bl = sorted(blocks, key=lambda b: -sum(i[2] for i in b))
    for b in bl[:top]:
        n = sum(i[2] for i in b)
        s = sum(i[3] for i in b)
        ops = Counter(i[1].split()[0].split(".")[0] if not i[1].startswith("@") else i[1].split()[1].split(".")[0]
                      for i in b)
        mix = " ".join(f"{k}:{v}" for k, v in ops.most_common(8))
        print(f"{hex(b[0][0])[-5:]}..{hex(b[-1][0])[-5:]} len {len(b):4d} x{b[0][2]:.3g} = {n / total * 100:5.1f}% "
              f"inst, {s / max(1, samples) * 100:5.1f}% stalls | {mix}")
        if show and b is not None and len(b) <= show:
            for i in b:
                print(f"      {hex(i[0])[-5:]} {i[1]}  [{i[3]}]")


if __name__ == "__main__":
    main()
