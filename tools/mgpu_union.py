"""Real multi-process check of the sharded path: under torchrun on N
GPUs, each rank all-gathers the length shards (NCCL), runs the global GPU FFD + device LPT, computes
attention fwd/bwd on ITS bins only, and the union of the per-rank outputs (gathered to rank 0) must
equal the single-GPU result bit for bit.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_union.py [out.json]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_11101_b200 import attention, dist as vdist, packing, synthetic  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    H, d, n_local = 8, 128, 200
    local = torch.from_numpy(synthetic.gen_lengths(n_local, synthetic.DIST_UNIFORM, 16, 512, seed=100 + rank)).to(dev)
    L_t = vdist.allgather_lengths(local)  # the path's only collective
    L = L_t.cpu().numpy()
    T = int(L.sum())
    plan = packing.pack_ffd(L_t, 8192)
    g = torch.Generator(device=dev).manual_seed(7)  # identical global tensors on every rank
    q, k, v, do = (torch.randn(T, H, d, device=dev, generator=g).bfloat16() for _ in range(4))
    src_off = np.concatenate([[0], np.cumsum(L)[:-1]])
    sp = vdist.shard_lpt(plan, world, rank)
    nseg = sp.nseg()
    ids = np.sort(sp.local_ids[:nseg].cpu().numpy())
    rows = torch.from_numpy(np.concatenate([src_off[i] + np.arange(L[i]) for i in ids])).to(dev)
    ql, kl, vl, dol = (x[rows].contiguous() for x in (q, k, v, do))
    cu = sp.local_cu[: nseg + 1]
    ol, lsel = attention.varlen_attn_fwd(ql, kl, vl, cu, seg_src=sp.local_seg_src[:nseg])
    res = (ol,) + attention.varlen_attn_bwd(dol, ql, kl, vl, ol, lsel, cu, seg_src=sp.local_seg_src[:nseg])
    # gather (rows, outputs) to every rank (padded all-gather)
    cnt = torch.tensor([rows.numel()], device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    mx = int(max(c.item() for c in cnts))
    def gather(x):
        pad = torch.zeros((mx,) + tuple(x.shape[1:]), dtype=x.dtype, device=dev)
        pad[: x.shape[0]] = x
        out = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(out, pad)
        return [o[: int(c.item())] for o, c in zip(out, cnts)]
    all_rows = gather(rows)
    outs = [gather(x) for x in res]
    ok = {}
    if rank == 0:
        seg = packing.seg_src(plan)
        o, lse = attention.varlen_attn_fwd(q, k, v, plan.cu_seqlens, seg_src=seg)
        full = (o,) + attention.varlen_attn_bwd(do, q, k, v, o, lse, plan.cu_seqlens, seg_src=seg)
        seen = torch.zeros(T, dtype=torch.bool, device=dev)
        for name, f, parts in zip(("o", "dq", "dk", "dv"), full, outs):
            got = torch.full_like(f, float("nan"))
            for r_, x in zip(all_rows, parts):
                got[r_] = x
                seen[r_] = True
            ok[name] = bool(torch.equal(got, f))
        ok["rows_disjoint_and_complete"] = bool(seen.all()) and sum(int(c.item()) for c in cnts) == T
        res_line = {"world": world, "tokens": T, "bins": plan.num_bins(), "bit_identical": ok}
        print(json.dumps(res_line), flush=True)
        if len(sys.argv) > 1:
            Path(sys.argv[1]).write_text(json.dumps(res_line) + "\n")
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not all(ok.values()):
        sys.exit(1)


if __name__ == "__main__":
    main()
