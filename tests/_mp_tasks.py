"""Picklable per-rank tasks for run_workers (spawned processes import this module)."""

import numpy as np

from paper_1811_11141_b200 import GradientBuffer, ring_allreduce


def sum_task(config, session):
    vals = np.arange(23, dtype="<f4") + config.rank
    buf = GradientBuffer(1, 1, vals)
    assert ring_allreduce(buf, config, session) is buf
    n = config.n_workers
    assert np.array_equal(buf.values, np.arange(23, dtype="<f4") * n + n * (n - 1) / 2)
    buf2 = GradientBuffer(1, 1, np.ones(5, dtype="<f4"))
    ring_allreduce(buf2, config, session)
    assert np.array_equal(buf2.values, np.full(5, n, dtype="<f4"))
    return session.counters.frames_sent


def single_element_task(config, session):
    buf = GradientBuffer(1, 1, np.array([float(config.rank + 1)], dtype="<f4"))
    ring_allreduce(buf, config, session)
    n = config.n_workers
    return bool(buf.values[0] == n * (n + 1) / 2)


def mismatched_task(config, session):
    size = 8 if config.rank == 0 else 12
    ring_allreduce(GradientBuffer(1, 1, np.zeros(size, dtype="<f4")), config, session)
    return True


def collective_task(config, session):
    verdicts = []
    for elements in (1, 17, 1_000_000, 5_000_003):
        buf = GradientBuffer(1, 1, np.full(elements, float(config.rank + 1), dtype="<f4"))
        ring_allreduce(buf, config, session)
        n = config.n_workers
        verdicts.append(bool((buf.values == n * (n + 1) / 2).all()))
    return verdicts


def random_task(config, session, *, arrays):
    """Reduce the golden per-rank inputs through the real IPC path."""
    import torch

    out = {}
    for key, vals in arrays[config.rank].items():
        buf = GradientBuffer(1, 1, vals.copy())
        ring_allreduce(buf, config, session)
        out[key] = buf.values.copy()
        t = torch.from_numpy(vals.copy()).to(session.device)
        ring_allreduce(GradientBuffer(1, 1, t), config, session)
        out[key + "_tensor"] = t.cpu().numpy()
    return out


def emulate_task(config, session, *, profile, plan, fused, graph):
    from paper_1811_11141_b200 import run_emulation

    return run_emulation(profile, plan, config, session, 3, warmup=1, fused=fused, graph=graph)
