"""One rank of tests/test_gpu_shard.py::test_shard_ipc_two_processes_one_gpu: the
one-process-per-GPU sharded path (IPC handles all-gathered over gloo, as bench.py does)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, out = int(sys.argv[1]), sys.argv[2]
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from oracle.oracle import Oracle
    from paper_2502_16949_b200 import Engine, ModelConfig, TrainConfig
    orc = Oracle("f32")
    n, r, d, batch = 1000, 6, 16, 200
    h, rel, t = orc.synthetic_train(n, r, 2400, 5)
    st = orc.init_store("transe", n, r, d, d, 5)
    cfg = ModelConfig.make("transe", d, d, "l2")
    eng = Engine(0)
    eng.store_upload(cfg, st.entity, st.relation)
    eng.set_triples(h, rel, t, n, r)
    eng.negative_sample(6)
    mine = eng.shard_export(rank, 2, batch)
    handles = [None, None]
    dist.all_gather_object(handles, mine)
    eng.shard_import(handles)
    tc = TrainConfig.make(lr=0.05, batch_size=batch, seed=6)
    losses = [eng.train_epoch(cfg, tc, ep, 0.05).loss for ep in range(2)]
    dist.barrier()
    ge, gr, _, _ = eng.store_download()
    np.savez(os.path.join(out, f"rank{rank}.npz"), entity=ge, relation=gr, loss=np.array(losses))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
