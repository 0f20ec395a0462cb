"""eta of one link over several GPUs of a node: each rank evaluates one cost-balanced shard of the
region list (isrs_egn_nli_shard), the per-COI sums are all-gathered, and every rank combines them
in fixed rank order (isrs_egn_combine) -> the same eta, bitwise, on every rank.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 examples/eta_multi_gpu.py c2
    (one rank per GPU, NCCL; `--backend gloo` runs the same logic with host-side collectives)
"""
import argparse
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_11614_b200 as isrs  # noqa: E402
from workloads import bj_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="c1")
    ap.add_argument("--backend", default="nccl")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if a.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(a.backend)
    link = bj_config(a.config)
    with isrs.Engine(link, device=local) as eng:
        sums = eng.nli_shard(rank, world)                              # [n_ch, 6], this rank's shard
        gathered = torch.empty(world * sums.numel(), dtype=sums.dtype, device=sums.device)
        dist.all_gather_into_tensor(gathered, sums.reshape(-1))
        eta = eng.combine(gathered.reshape(world, *sums.shape))       # fixed rank order
        pts, pspans, nreg = eng.work()
    eta_db = (10 * torch.log10(eta)).cpu().tolist()
    print(f"rank {rank}/{world}: {nreg} regions, {pspans} point-spans in this shard; "
          f"eta[dB] first/mid/last = {eta_db[0]:.6f} {eta_db[len(eta_db) // 2]:.6f} {eta_db[-1]:.6f}",
          flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
