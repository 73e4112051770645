"""Empirical parametrization on this B200 box, then a prediction.

torchrun --nproc-per-node N tools/calibrate_b200.py OUT.json
  * every rank: NCCL Allreduce times over message sizes 64 KiB..256 MiB for the whole group
    and (N >= 4) for the sub-group of ranks {0, 1}; ring-form least-squares alpha/beta per
    group size (one system tier per size);
  * rank 0: per-layer forward / backward times of ResNet-50 at b = 32 (torch / cuDNN,
    fp32 with the default TF32 convolutions), turned into an effective-FLOP layer table;
  * rank 0: the cfg2 strategy sweep (six strategies x b, one alpha/beta row = the measured
    tiers) over the calibrated system through the CUDA library: the best configurations
    for training ResNet-50 on these N GPUs, per the calibrated model.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from workloads import calibrate as CAL
from workloads import models as M
from workloads import sweeps as W


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/calibration.json"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ws, rank = dist.get_world_size(), dist.get_rank()
    sizes = [1 << e for e in range(16, 29, 2)]
    tiers = []
    if ws >= 4:
        g2 = dist.new_group([0, 1])
        if rank in (0, 1):
            tiers.append(CAL.calibrate_tier(sizes, reps=20, group=g2))
        dist.barrier()
    tiers.append(CAL.calibrate_tier(sizes, reps=20))
    # per-pattern parameters (SURVEY f2 / DESIGN.md Q40): small-message tree fit and its
    # crossing with the ring form, point-to-point ping-pong (ranks 0, 1), ring Allgather
    small = [1 << e for e in range(10, 19)]
    t_small = CAL.time_allreduce(small, reps=20)
    tree = CAL.fit_allreduce_tree(ws, small, t_small, k=1)
    ring = (tiers[-1]["alpha_s"], tiers[-1]["beta_s_per_B"])
    thr = CAL.tree_threshold(ws, ring, tree[:2], k=1)
    t_p2p = CAL.time_p2p(sizes, reps=20)
    p2p = CAL.fit_p2p(sizes, t_p2p)
    ka, kb = CAL.p2p_scales(tiers[-1], p2p[:2])
    t_ag = CAL.time_allgather([m // ws for m in sizes], reps=20)
    ag = CAL.fit_allgather(ws, [m // ws for m in sizes], t_ag)
    patterns = {"tree_alpha_s": tree[0], "tree_beta_s_per_B": tree[1], "tree_fit_rms_rel": tree[2],
                "tree_threshold_B": thr, "small_sizes_B": small, "small_allreduce_s": t_small,
                "p2p_alpha_s": p2p[0], "p2p_beta_s_per_B": p2p[1], "p2p_fit_rms_rel": p2p[2],
                "p2p_alpha_scale": ka, "p2p_beta_scale": kb, "p2p_s": t_p2p,
                "allgather_alpha_s": ag[0], "allgather_beta_s_per_B": ag[1], "allgather_fit_rms_rel": ag[2],
                "allgather_s": t_ag}
    if rank == 0:
        m = M.resnet(50)
        times = CAL.time_layers(m, b=32, reps=10)
        R_ref = 1e15
        em = CAL.empirical_model(m, times, R_ref)
        sysm = CAL.system_from_tiers(tiers, flops_per_s=R_ref, hbm_bytes=180 * W.GiB, tree_threshold=thr,
                                     tree_chunks=1, p2p_alpha_scale=ka, p2p_beta_scale=kb)
        import paper_2104_09075_b200 as P
        sw = W.config2(n_alpha=1, n_beta=1, pipe_smax=min(4, ws))
        sw.models = [em]
        sw.system = sysm
        for sb in sw.subs:   # measured tiers only: one alpha/beta row
            sb.alpha, sb.beta = [], []
            sb.dims = [d for d in sb.dims if d[0] * d[1] * d[2] * d[3] <= ws]
        sw.subs = [sb for sb in sw.subs if sb.dims or sb.family == W.PIPELINE]
        ctx = P.Context(local)
        spec = ctx.prepare(sw)
        hits, nf = ctx.topk(spec, 10)
        best = []
        for idx, key in hits:
            if idx == 2 ** 64 - 1:
                continue
            c = ctx.decode(spec, idx)
            pr = ctx.explain(spec, idx)
            best.append({"idx": idx, "family": W.FAMILY_NAMES[c.family], "b": c.b, "B": c.B, "p": c.p,
                         "dims": list(c.dims), "S": c.S, "stages": list(c.stage_end[:c.n_stages]),
                         "t_iter_s": pr.t_iter, "t_epoch_s": pr.t_epoch, "mem_GB": pr.mem / 1e9})
        rows = [{"name": r.name, "fw_s_per_sample": t[0], "bw_s_per_sample": t[1]}
                for r, t in zip(m.layers, times) if t is not None]
        res = {"world_size": ws, "device": torch.cuda.get_device_name(local), "tiers": tiers, "patterns": patterns,
               "resnet50_layers_b32": rows, "effective_flops_per_s": em.meta["effective_flops_per_s"],
               "prediction": {"sweep": "cfg2 strategies on the calibrated system", "configs": ctx.sweep_size(spec),
                              "feasible": nf, "top": best}}
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps({k: res[k] for k in ("world_size", "device", "effective_flops_per_s")}))
        for t in tiers:
            print(f"tier p={t['p']}: alpha {t['alpha_s']*1e6:.2f} us, 1/beta {1/t['beta_s_per_B']/1e9:.1f} GB/s, rms {t['fit_rms_rel']:.3f}")
        for b_ in best[:5]:
            print(b_)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
