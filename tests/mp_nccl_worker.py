"""Worker of tests/test_tp_nccl_gpu.py (one process per GPU, launched by torch.distributed.run): the
real NCCL tensor-parallel path of libsirius on Llama-3-8B layer shapes (2 layers, full vocab).  Every
rank bootstraps the communicator (paper_2409_03856_b200/tp.py), uploads its own shard and runs the
Sirius loop; rank 0 checks the tokens and per-kernel advances against the CPU oracle at TP 1 (the
global active set is the disjoint union of the per-rank sets, reading D1) and prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2409_03856_b200 import driver, sirius as S, tp as TP  # noqa: E402
from synth import gpu as sg  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    comm = TP.nccl_bootstrap(S.load(), world, rank)
    cfg = synth.LLAMA3_8B_2L
    thr = synth.layer_thresholds(cfg, 0.5)
    prompt = synth.eval_prompt(cfg, 0, 128)
    ctx = S.Sirius(cfg, sg.device_weights(cfg, world, rank), thr, batch=1, max_seq=256, max_gamma=16,
                   tp_size=world, tp_rank=rank, nccl_comm=comm)
    par = os.environ.get("SIRIUS_TEST_PAR", "0") == "1"
    if par:  # fused NVLink peer all-reduce of the decode step (CUDA-IPC mapped comm buffers)
        TP.par_bootstrap(ctx)
    out = driver.Driver(ctx).sirius([prompt], 48, 16, 0.3)
    res = {"rank": rank, "tokens": out.tokens[0], "advances": out.advances(0)}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        from oracle import sirius_oracle as so
        ref = so.generate(so.OracleModel(cfg, synth.host_weights(cfg), max_seq=256, max_gamma=16), prompt, 48, 16,
                          0.3, thr)
        ok = all(r["tokens"] == ref.tokens for r in allres) and \
            all(r["advances"] == ref.advances[:len(r["advances"])] for r in allres)
        print(json.dumps({"world": world, "par": par, "ok": ok, "tokens_equal_across_ranks":
                          all(r["tokens"] == allres[0]["tokens"] for r in allres)}), flush=True)
        if not ok:
            sys.exit(1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
