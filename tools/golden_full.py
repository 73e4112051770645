"""Whole-sweep oracle goldens: top-64 (idx, key) and feasible count of a full BASELINE config.

    python tools/golden_full.py CFG [--threads N] [--chunk-log2 L]

Calls only `oracle/` (the CPU checker) and `workloads/` (the input generator): no value
here comes from the CUDA path.  The sweep is cut into chunks of 2^L consecutive indices;
each chunk's top-64 + count is appended to a checkpoint (tests/golden/full_cfgN.partial.jsonl,
git-ignored), so a long run (cfg5: ~8 h on 8 cores) survives interruption.  When every chunk is
done the chunks are merged -- the top-64 of a union is the top-64 of the per-chunk top-64
lists under the lexicographic (key, idx) order -- and written to
tests/golden/full_cfgN.json with keys as exact float.hex strings.

Cites: PAPER.md P:706 (§5.2) "all the permutations of possible configurations" and
P:429 "suggesting the best strategy" -- the whole-sweep reduction the GPU path computes.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

K = 64
UMAX = (1 << 64) - 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--chunk-log2", type=int, default=30)
    ap.add_argument("--stride", type=int, default=1,
                    help="evaluate every stride-th chunk only (sampled chunks; no whole-sweep merge)")
    ap.add_argument("--reverse", action="store_true", help="evaluate the chunks from the last one down")
    ap.add_argument("--time-budget", type=float, default=0.0, help="stop starting chunks after this many seconds")
    ap.add_argument("--out", default="", help="checkpoint file (default tests/golden/full_cfgN.partial.jsonl)")
    ap.add_argument("--merge-only", action="store_true",
                    help="no evaluation: merge every tests/golden/full_cfgN*.jsonl checkpoint (deduplicated by "
                         "chunk) into full_cfgN.chunks.jsonl, and into full_cfgN.json when every chunk is there")
    args = ap.parse_args()

    from oracle import oracle as O
    from workloads import sweeps as W
    sw = W.CONFIGS[args.cfg]()
    osw = O.OracleSweep(sw)
    n = osw.size()
    chunk = 1 << args.chunk_log2
    gdir = os.path.join(ROOT, "tests", "golden")
    part = args.out or os.path.join(gdir, f"full_cfg{args.cfg}.partial.jsonl")
    done = {}
    import glob
    for path in sorted(set(glob.glob(os.path.join(gdir, f"full_cfg{args.cfg}*.jsonl")) + [part])):
        if not os.path.exists(path):
            continue
        for ln in open(path):
            r = json.loads(ln)
            if r["n"] == n and r["chunk"] == chunk:
                done[r["first"]] = r
    firsts = list(range(0, n, chunk))[::args.stride]
    if args.reverse:
        firsts = firsts[::-1]
    t_all = time.time()
    if args.merge_only:
        with open(os.path.join(gdir, f"full_cfg{args.cfg}.chunks.jsonl"), "w") as f:
            for a in sorted(done):
                f.write(json.dumps(done[a]) + "\n")
        print(f"merged {len(done)} of {len(firsts)} chunks")
        if len(done) < len(firsts):
            return
    with open(part, "a") as f:
        for a in firsts:
            if a in done:
                continue
            if args.time_budget and time.time() - t_all > args.time_budget:
                break
            c = min(chunk, n - a)
            t0 = time.time()
            hits, nf = osw.topk(a, c, K, nthreads=args.threads)
            r = {"n": n, "chunk": chunk, "first": a, "count": c, "n_feasible": nf,
                 "hits": [[int(i), float(k).hex()] for i, k in hits if i != UMAX],
                 "seconds": time.time() - t0, "threads": args.threads}
            f.write(json.dumps(r) + "\n")
            f.flush()
            done[a] = r
            print(f"cfg{args.cfg} chunk {len(done)}/{len(firsts)} [{a}, +{c}) {r['seconds']:.1f} s", flush=True)
    if args.stride > 1:
        print(f"sampled chunks done: {len(done)} (every {args.stride}-th of {len(range(0, n, chunk))})")
        return
    if len(done) < len(firsts):
        print(f"{len(done)} of {len(firsts)} chunks done; no whole-sweep file yet")
        return
    cand = []
    for r in done.values():
        cand += [(float.fromhex(k), i) for i, k in r["hits"]]
    cand.sort()
    top = cand[:K]
    nf = sum(r["n_feasible"] for r in done.values())
    out = {"_about": "Whole-sweep top-64 and feasible count written by tools/golden_full.py from the CPU "
                     "oracle only (oracle/oracle.c); keys = t_epoch in seconds as float.hex. "
                     "PAPER.md P:706 (all permutations), P:429 (best strategy); order (key, idx), Q32.",
           "workload": sw.name, "configs": n, "k": K, "n_feasible": nf,
           "hits": [[i, k.hex()] for k, i in top],
           "oracle_chunk_seconds_sum": round(sum(r["seconds"] for r in done.values()), 1),
           "oracle_runs": "chunked; threads per chunk in the checkpoint records"}
    path = os.path.join(gdir, f"full_cfg{args.cfg}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {path}: {nf} feasible, best idx {top[0][1] if top else None} ({time.time() - t_all:.0f} s)")


if __name__ == "__main__":
    main()
