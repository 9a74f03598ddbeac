"""Row-sharded data parallel (shard.cu) on one B200: G contexts on device 0
form one group (the same kernels, plans and peer-flag barriers a G-GPU run uses; peer
pointers are plain device pointers here). A G-rank run must equal the single-device
oracle at batch_size = global batch (training.cpp:82-92): tables bit for bit, losses
within 1e-5 (the shard losses are summed per rank)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_2502_16949_b200 import Engine, EngineError, ModelConfig, TrainConfig

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _group(world, cfg, st, h, rel, t, n, r, seed, batch):
    engines = [Engine(0) for _ in range(world)]
    for e in engines:
        e.store_upload(cfg, st.entity, st.relation)
        e.set_triples(h, rel, t, n, r)
        e.negative_sample(seed)
    Engine.shard_group_init(engines, batch)
    return engines


@pytest.mark.parametrize("world,model,norm,d,m_extra", [(2, "transe", "l2", 32, 0), (4, "transe", "l2", 64, 3),
                                                        (4, "transe", "l1", 16, 0), (2, "toruse", "l2", 32, 5),
                                                        (4, "toruse", "l1", 8, 0), (2, "transe", "l2", 256, 7)])
def test_shard_group_matches_oracle_bitwise(orc32, world, model, norm, d, m_extra):
    n, r, batch = 1501, 31, 1000  # ranks own different entity / relation counts
    h, rel, t = orc32.synthetic_train(n, r, 12000, 2)
    if m_extra:  # a ragged last batch whose shards are uneven
        h, rel, t = (np.concatenate([a, a[:m_extra]]) for a in (h, rel, t))
    st = orc32.init_store(model, n, r, d, d, 2)
    cfg = ModelConfig.make(model, d, d, norm)
    engines = _group(world, cfg, st, h, rel, t, n, r, 9, batch)
    tc = TrainConfig.make(lr=0.05, batch_size=batch, seed=9)
    losses = []
    for ep in range(3):
        reps = Engine.shard_group_train_epoch(engines, cfg, tc, ep, 0.05)
        assert len({x.loss for x in reps}) == 1  # every rank reports the same global loss
        losses.append(reps[0].loss)
    ro = orc32.fit(model, st, h, rel, t, orc32.train_config(epochs=3, lr=0.05, batch_size=batch, seed=9), norm=norm)
    for a, b in zip(losses, ro):
        assert abs(a - b.loss) <= 1e-5 * max(1.0, abs(b.loss)), (a, b.loss)
    for e in engines:  # download gathers every rank's shard: identical on all ranks
        ge, gr, _, _ = e.store_download()
        assert np.array_equal(gr, st.relation)
        assert np.array_equal(ge, st.entity)
    for e in engines:
        e.close()


def test_shard_group_non_finite_loss_stops_every_rank(orc32):
    """A NaN entity row makes one shard's loss non-finite: every rank raises the
    reference's TrainingError for the same batch, with nothing applied from it on."""
    n, r, d, batch, world = 800, 10, 16, 400, 2
    h, rel, t = orc32.synthetic_train(n, r, 5000, 3)
    st = orc32.init_store("transe", n, r, d, d, 3)
    st.entity[int(h[-1])] = np.nan
    cfg = ModelConfig.make("transe", d, d, "l2")
    engines = _group(world, cfg, st, h, rel, t, n, r, 4, batch)
    tc = TrainConfig.make(lr=0.05, batch_size=batch, seed=4)
    with pytest.raises(EngineError) as e:
        Engine.shard_group_train_epoch(engines, cfg, tc, 0, 0.05)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as o:
        orc32.fit("transe", st, h, rel, t, orc32.train_config(epochs=1, lr=0.05, batch_size=batch, seed=4))
    assert e.value.kind == "TrainingError" and e.value.msg in str(o.value), (e.value.msg, str(o.value))
    ge = engines[1].store_download()[0]
    ok = ~np.isnan(st.entity).any(axis=1)
    assert np.array_equal(ge[ok], st.entity[ok])  # the batches before the failing one, as the reference
    for x in engines:
        x.close()


def test_shard_config_errors(orc32):
    n, r, d = 1200, 9, 8
    h, rel, t = orc32.synthetic_train(n, r, 6000, 1)
    st = orc32.init_store("transe", n, r, d, d, 1)
    cfg = ModelConfig.make("transe", d, d, "l2")
    engines = [Engine(0) for _ in range(8)]
    for e in engines:
        e.store_upload(cfg, st.entity, st.relation)
        e.set_triples(h, rel, t, n, r)
        e.negative_sample(1)
    with pytest.raises(EngineError) as e:  # world must be a power of two up to 8
        Engine.shard_group_init(engines[:3], 300)
    assert e.value.kind == "ConfigError"
    with pytest.raises(EngineError) as e:  # at most 4 ranks share one device
        Engine.shard_group_init(engines, 400)
    assert e.value.kind == "ConfigError"
    with pytest.raises(EngineError) as e:  # global batch must split evenly
        Engine.shard_group_init(engines[:2], 301)
    assert e.value.kind == "ConfigError"
    Engine.shard_group_init(engines[:2], 300)
    with pytest.raises(EngineError) as e:  # the batch the plan buffers were sized for
        Engine.shard_group_train_epoch(engines[:2], cfg, TrainConfig.make(batch_size=200, seed=1), 0, 0.01)
    assert e.value.kind == "ConfigError"
    for x in engines:
        x.close()


def test_shard_ipc_two_processes_one_gpu(orc32, tmp_path):
    """The one-process-per-GPU path (skg_shard_export / IPC handles / skg_shard_import,
    skg_train_epoch with barriers across processes), both processes on device 0.
    Kernels of two processes time-slice on one GPU, so every barrier waits for the
    peer's time slice: tiny shapes only."""
    port = socket.socket()
    port.bind(("127.0.0.1", 0))
    p = port.getsockname()[1]
    port.close()
    script = os.path.join(ROOT, "tests", "shard_ipc_worker.py")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(p), WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, script, str(k), str(tmp_path)], env=dict(env, RANK=str(k)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for k in range(2)]
    outs = [pr.communicate(timeout=600)[0] for pr in procs]
    assert all(pr.returncode == 0 for pr in procs), outs
    n, r, d, batch = 1000, 6, 16, 200
    h, rel, t = orc32.synthetic_train(n, r, 2400, 5)
    st = orc32.init_store("transe", n, r, d, d, 5)
    ro = orc32.fit("transe", st, h, rel, t, orc32.train_config(epochs=2, lr=0.05, batch_size=batch, seed=6))
    for k in range(2):
        got = np.load(os.path.join(tmp_path, f"rank{k}.npz"))
        assert np.array_equal(got["entity"], st.entity) and np.array_equal(got["relation"], st.relation)
        for a, b in zip(got["loss"], ro):
            assert abs(a - b.loss) <= 1e-5 * max(1.0, abs(b.loss))
