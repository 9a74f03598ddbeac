"""CPU tests of the `kge train` artifact writers (skg_run_log_*, tools/kge.cpp:181-247):
the files must read like the reference CLI's: train_log.jsonl compact records with
sorted keys (nlohmann::json objects are std::maps) flushed per epoch, loss.log with
%.17g losses, summary.json as dump(2). Restates test_cli.cpp:139-182 (JSONL and
loss.log agreement, byte-identical artifacts across reruns)."""
import json
import os

import numpy as np

from paper_2502_16949_b200.engine import EpochReport, ModelConfig, RunLog, RunSummary, TrainConfig


def _reps():
    out = []
    for e, loss in enumerate([0.515363395, 0.25, 1e-05, 123456.75]):
        r = EpochReport()
        r.epoch, r.loss = e, float(np.float32(loss))
        r.t_forward_s, r.t_backward_s, r.t_step_s = 0.001 * (e + 1), 0.5, 0.0
        out.append(r)
    return out


def _write(d):
    lg = RunLog(str(d))
    reps = _reps()
    for r in reps:
        lg.epoch(r)
    cfg = ModelConfig.make("transe", 16, 16, "l2")
    tc = TrainConfig.make(lr=4e-4, margin=0.5, epochs=4, batch_size=32, seed=7, scheduler=(10, 0.5))
    info = RunSummary(b"sparse", b"synthetic", 1000, 20, 4500, 250, 250, 0, 0, 8, 4, reps[-1].loss,
                      sum(r.t_forward_s for r in reps), sum(r.t_backward_s for r in reps), 0.0, None)
    lg.summary(cfg, tc, info)
    lg.close()
    return reps


def test_jsonl_and_loss_log_match_the_reference_format(tmp_path):
    reps = _write(tmp_path)
    lines = open(tmp_path / "train_log.jsonl").read().splitlines()
    assert len(lines) == 4
    for line, r in zip(lines, reps):
        rec = json.loads(line)
        # compact nlohmann dump: sorted keys, no spaces, shortest round-trip doubles
        assert line == json.dumps(rec, sort_keys=True, separators=(",", ":"))
        assert list(rec) == ["epoch", "loss", "t_backward_s", "t_forward_s", "t_step_s"]
        assert rec["epoch"] == r.epoch and rec["loss"] == float(np.float32(r.loss))
    losses = open(tmp_path / "loss.log").read().splitlines()
    for line, r in zip(losses, reps):  # kge.cpp:32-36: "%.17g"
        e, v = line.split()
        assert int(e) == r.epoch and v == "%.17g" % float(np.float32(r.loss))
        assert float(v) == json.loads(lines[r.epoch])["loss"]  # test_cli.cpp:139-171 agreement


def test_summary_json_layout(tmp_path):
    _write(tmp_path)
    text = open(tmp_path / "summary.json").read()
    s = json.loads(text)
    assert text == json.dumps(s, sort_keys=True, indent=2) + "\n"  # nlohmann dump(2) layout
    assert s["model"] == "transe" and s["norm"] == "l2" and s["engine"] == "sparse"
    assert s["config"]["scheduler"] == {"every_epochs": 10, "factor": 0.5}
    assert s["config"]["seed"] == 7 and s["config"]["threads"] == 8
    assert s["config"]["lr"] == float(np.float32(4e-4))  # Real lr stored as double, like the REAL32 build
    m = 4500
    assert s["flops"]["per_epoch_estimate"] == 4 * 3 * m * 16 * 2  # kge.cpp:146-160 (TransE: spmm + norms)
    assert s["artifacts"]["log"].endswith("train_log.jsonl") and s["artifacts"]["checkpoint"].endswith("checkpoint.bin")
    assert s["time"]["total_s"] == s["time"]["forward_s"] + s["time"]["backward_s"]


def test_artifacts_are_byte_identical_across_reruns(tmp_path):  # test_cli.cpp:173-182
    _write(tmp_path / "a")
    _write(tmp_path / "b")
    for f in ("train_log.jsonl", "loss.log"):
        assert open(tmp_path / "a" / f).read() == open(tmp_path / "b" / f).read()


def test_logs_append_like_the_cli(tmp_path):  # kge.cpp:189-190 open in append mode
    _write(tmp_path)
    _write(tmp_path)
    assert len(open(tmp_path / "train_log.jsonl").read().splitlines()) == 8
