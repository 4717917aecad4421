"""N>1 plumbing on CPU: two gloo ranks run the replica bookkeeping the bench
uses over NCCL (barrier, max-over-ranks time, summed units, per-rank
streams), and each replica runs a short CPU checker stream of its own."""
import json
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
mp = pytest.importorskip("torch.multiprocessing")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    from paper_2308_16395_b200 import datagen as dg, replicas
    import py_oracle

    g = replicas.init("gloo")
    cfg = replicas.stream_config(dg.scaled(dg.CONFIGS["c2"], (12, 10, 8), n_slices=8, n_init=3), g.rank)
    gen = dg.TuckerStream(cfg)
    chk = py_oracle.load_oracle()
    x = gen.init_numpy().reshape(gen.init_dims()[::-1]).transpose()
    h = chk.stream_init(x, cfg.tau)
    steps = 4
    for t in range(steps):
        h.update_flat(gen.slice_numpy(cfg.n_init + t))
    replicas.barrier(g)
    fake_seconds = 1.0 + g.rank  # the slower rank sets the job time
    rate, tmax = replicas.job_rate(g, float(steps), fake_seconds)
    st = h.export()
    rec = {"rank": g.rank, "world": g.world, "rate": rate, "tmax": tmax, "seed": cfg.seed,
           "core0": float(np.asarray(st.core).ravel()[0]), "n_d": int(st.n_d)}
    with open(os.path.join(out_dir, f"rank{g.rank}.json"), "w") as f:
        json.dump(rec, f)
    replicas.close(g)


def test_two_gloo_replicas(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    recs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    for r in recs:
        assert r["world"] == world
        assert r["tmax"] == pytest.approx(2.0)             # max over ranks
        assert r["rate"] == pytest.approx(2 * 4 / 2.0)     # summed units / slowest rank
        assert r["n_d"] == 3 + 4
    assert recs[0]["seed"] != recs[1]["seed"]               # independent streams
    assert recs[0]["core0"] != recs[1]["core0"]


def test_single_process_group_defaults(monkeypatch):
    from paper_2308_16395_b200 import replicas
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    g = replicas.init("gloo")
    assert (g.world, g.rank) == (1, 0)
    assert replicas.job_rate(g, 10.0, 2.0) == (5.0, 2.0)
