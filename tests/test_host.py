"""Host-side logic (no GPU): tiling / index sets, schedules and configs, problem
generator, phi family, and the multi-process replica reduction of bench.py.

The tiling tests mirror the reference's own (`pkg/tests/test_schwarz.py:43-126`).
"""

import hashlib
import os
import socket

import numpy as np
import pytest

import raspen_oracle as O
from paper_2411_00546_b200 import (ContinuationSchedule, Grid, KrylovConfig, NewtonConfig,
                                   NonfiniteFieldError, decompose, make_phi)
from paper_2411_00546_b200.problems import CONFIGS, build_fields
from paper_2411_00546_b200.schwarz import _tile_edges
from paper_2411_00546_b200.system import Cubic, ExpMinusOne, Nonlinearity, smoothed_projection


class TestTiling:
    def test_even_split_and_remainder(self):
        assert _tile_edges(8, 2) == [(0, 4), (4, 8)]
        assert _tile_edges(9, 2) == [(0, 4), (4, 9)]
        assert _tile_edges(17, 3) == [(0, 5), (5, 10), (10, 17)]
        assert _tile_edges(2047, 64)[-1] == (1953, 2047)

    def test_errors(self):
        with pytest.raises(ValueError, match="nonempty"):
            _tile_edges(3, 4)
        with pytest.raises(ValueError, match="row direction"):
            decompose(Grid(8), 2, 1, 5)
        with pytest.raises(ValueError, match="column direction"):
            decompose(Grid(8), 1, 2, 5)
        with pytest.raises(ValueError, match="at least one tile"):
            decompose(Grid(8), 0, 2, 1)
        with pytest.raises(ValueError, match="nonnegative"):
            decompose(Grid(8), 2, 2, -1)
        decompose(Grid(8), 1, 1, 99)

    def test_corner_block_and_clipping(self):
        dec = decompose(Grid(8), 2, 2, 2)
        sub = dec.subdomains[0]
        assert sub.rows == (0, 6) and sub.cols == (0, 6) and sub.size == 36
        assert sub.idx[5] == 5 and sub.idx[6] == 8
        np.testing.assert_array_equal(sub.idx[sub.own_in_local], sub.own)
        assert decompose(Grid(8), 2, 2, 3).subdomains[3].rows == (1, 8)

    @pytest.mark.parametrize("s1,s2", [(1, 1), (2, 2), (2, 3), (3, 3)])
    @pytest.mark.parametrize("n", [8, 9, 17])
    def test_ownership_partition_and_scatter(self, s1, s2, n):
        dec = decompose(Grid(n), s1, s2, 2)
        owned = np.concatenate([s.own for s in dec.subdomains])
        np.testing.assert_array_equal(np.sort(owned), np.arange(n * n))
        x = np.random.default_rng(5).standard_normal(2 * n * n)
        out = np.zeros_like(x)
        for s in dec.subdomains:
            out[s.pair_own] = x[s.pair_idx][s.pair_own_in_local]
        np.testing.assert_array_equal(out, x)

    @pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4", "cfg5"])
    def test_matches_oracle_decomposition(self, name):
        cfg = CONFIGS[name]
        dec = decompose(Grid(cfg.n), cfg.s1, cfg.s2, cfg.overlap)
        rects = O.decompose(cfg.n, cfg.s1, cfg.s2, cfg.overlap)
        assert len(dec) == len(rects) == cfg.s1 * cfg.s2
        for a, b in zip(dec.subdomains, rects):
            assert (a.rows, a.cols, a.own_rows, a.own_cols) == (b.rows, b.cols, b.own_rows, b.own_cols)

    def test_config5_is_ragged_as_written(self):
        cfg = CONFIGS["cfg5"]
        dec = decompose(Grid(cfg.n), cfg.s1, cfg.s2, cfg.overlap)
        shapes = {(s.rows[1] - s.rows[0], s.cols[1] - s.cols[0]) for s in dec.subdomains}
        assert (96, 96) in shapes and (33, 33) in shapes and len(shapes) == 9


class TestSchedulesAndConfigs:
    def test_schedule(self):
        with pytest.raises(ValueError):
            ContinuationSchedule(eps0=1e-12, eps_min=1e-10)
        with pytest.raises(ValueError):
            ContinuationSchedule(gamma=0.0)
        s = ContinuationSchedule.fixed(1e-3)
        assert s.eps0 == s.eps_min == 1e-3 and s.next_eps(1e-3) == 1e-3

    @pytest.mark.parametrize("eps_min,updates", [(1e-6, 7), (1e-7, 8)])
    def test_eps_path_float_drift(self, eps_min, updates):
        """1 -> 1e-6 by 0.1 takes 7 updates (1.0000000000000004e-06 -> 1e-06), SURVEY 0.12."""
        s = ContinuationSchedule(1.0, 0.1, eps_min)
        eps, k = 1.0, 0
        while eps != eps_min:
            eps = s.next_eps(eps)
            k += 1
        assert k == updates

    def test_config_validation(self):
        with pytest.raises(ValueError):
            NewtonConfig(tol=0.0)
        with pytest.raises(ValueError):
            NewtonConfig(sigma=0.5)
        with pytest.raises(ValueError):
            KrylovConfig(rel_tol=0.0, abs_tol=0.0)
        with pytest.raises(ValueError):
            KrylovConfig(max_iters=0)


class TestProblems:
    def test_generator_is_deterministic(self):
        for name in ("cfg2", "cfg3"):
            f1, y1 = build_fields(CONFIGS[name])
            f2, y2 = build_fields(CONFIGS[name])
            np.testing.assert_array_equal(f1, f2)
            np.testing.assert_array_equal(y1, y2)

    @pytest.mark.parametrize("name,digest", [
        ("cfg1", "2ebaf4c5d31768db"), ("cfg2", "e4bc46ff283c38da"), ("cfg3", "de4042620c68dbb8"),
        ("cfg4", "933272b9d0a04220"), ("cfg5", "5ec2e2af4e430391")])
    def test_generator_digests_are_frozen(self, name, digest):
        """The input convention of SURVEY 8d is frozen: the golden fixtures were
        generated from exactly these arrays (sha256 of f || y_d)."""
        f, yd = build_fields(CONFIGS[name])
        h = hashlib.sha256(np.ascontiguousarray(f).tobytes() + np.ascontiguousarray(yd).tobytes())
        assert h.hexdigest()[:16] == digest

    def test_baseline_shapes(self):
        assert CONFIGS["cfg4"].unknowns == 2 * 1023 * 1023
        assert (CONFIGS["cfg4"].s1, CONFIGS["cfg4"].overlap) == (16, 8)
        f3, _ = build_fields(CONFIGS["cfg3"])
        assert np.abs(f3).max() > 0


class TestPhi:
    def test_formulas(self):
        s = np.linspace(-3, 3, 101)
        c = Cubic()
        np.testing.assert_array_equal(c.value(s), s * s * s)
        np.testing.assert_array_equal(c.derivative(s), 3.0 * s * s)
        e = ExpMinusOne()
        np.testing.assert_allclose(e.value(s), np.expm1(s), rtol=1e-12, atol=1e-15)
        k = Nonlinearity(0.1)
        np.testing.assert_allclose(k.value(s), 0.1 * (s ** 3 + np.exp(0.1 * s)))
        assert make_phi("cubic").kind == 1 and make_phi("expm1").kind == 2

    def test_overflow_checks(self):
        with pytest.raises(NonfiniteFieldError):
            ExpMinusOne().derivative(np.array([0.0, 800.0]))
        assert np.isfinite(ExpMinusOne().value(np.array([800.0]), check=False)).all()

    def test_projection(self):
        x = np.linspace(-3, 3, 61)
        np.testing.assert_array_equal(smoothed_projection(x, 0.0), np.clip(x, -1, 1))
        assert np.all(np.abs(smoothed_projection(x, 1e-4) - np.clip(x, -1, 1)) <= 1e-2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _replica_worker(rank, world, port, out):
    import torch.distributed as td
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    d = bench.Dist("gloo")
    ms = d.max(100.0 + 10.0 * rank)        # slowest rank's time
    tot = d.sum(1000.0 * (rank + 1))       # all ranks' DOF-updates
    d.barrier()
    out[rank] = (ms, tot, tot / (ms / 1e3))
    d.close()


def test_bench_replica_reduction_gloo_world2():
    """bench.py N>1 path: max-over-ranks time, summed work (replicas, weak scaling)."""
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_replica_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1]
    ms, tot, val = out[0]
    assert ms == 110.0 and tot == 3000.0 and val == pytest.approx(3000.0 / 0.11)


def test_buffer_pools_retire_to_the_process_cache(monkeypatch):
    """Engine teardown hands cached device buffers to the process-wide
    retired cache (reused by size by the next engine, bounded, thread-safe);
    nothing here touches a device: _raw_free is replaced by a recorder."""
    from paper_2411_00546_b200 import _native as nat
    freed = []
    monkeypatch.setattr(nat, "_raw_free", lambda addr: freed.append(addr))
    monkeypatch.setattr(nat, "_RETIRED", nat._RetiredCache(limit_bytes=3 << 20))
    a = nat.BufferPool()
    a.give(0x1000, 1 << 20)
    a.give(0x2000, 1 << 20)
    a.give(0x3000, 2 << 20)
    a.release_all()                      # engine A torn down (its stream idle)
    assert freed == [0x3000] and nat._RETIRED.cached == 2 << 20   # the 2 MB one exceeds the limit
    b = nat.BufferPool()
    got = b.take(1 << 20)                # engine B reuses a retired buffer of that size
    assert got in (0x1000, 0x2000)
    assert b.take(5 << 20) is None       # no buffer of that size: caller allocates
    nat._RETIRED.give(0x4000, 4 << 20)   # over the cache limit: freed at once
    assert 0x4000 in freed
    nat.empty_cache()
    assert nat._RETIRED.cached == 0
    assert sorted(freed) == sorted([0x3000, 0x4000, 0x1000 if got == 0x2000 else 0x2000])


def test_retired_cache_give_never_blocks_on_its_own_lock():
    """A garbage-collection finalizer can run inside _RetiredCache.take / give while the
    thread holds the cache lock (Engine teardown -> release_all -> give): give must not
    block (it deadlocked the GPU suite against itself); the parked buffer is filed by
    the next caller."""
    from paper_2411_00546_b200 import _native as nat
    c = nat._RetiredCache(limit_bytes=1 << 20)
    c.give(0x1000, 256)
    assert c.take(256) == 0x1000 and c.take(256) is None
    assert c.lock.acquire(blocking=False)       # "inside take()" on this thread
    try:
        c.give(0x2000, 512)                     # re-entrant give: returns at once
    finally:
        c.lock.release()
    assert c.cached == 0 and c._pending == [(0x2000, 512)]
    assert c.take(512) == 0x2000                # filed and handed out by the next take
    assert c.cached == 0 and not c._pending


def test_retired_cache_survives_finalizers_during_take():
    """Finalizers that give buffers back run at arbitrary allocation points: force a
    collection from inside the locked region of take() through a dict subclass."""
    import gc
    from paper_2411_00546_b200 import _native as nat
    c = nat._RetiredCache(limit_bytes=1 << 20)

    class Victim:
        def __del__(self):
            c.give(0x3000, 1024)

    class Probe(dict):
        def get(self, k, d=None):
            v = Victim()
            v.loop = v          # a cycle: only the collector frees it
            del v
            gc.collect()        # the finalizer runs here, with c.lock held by take()
            return dict.get(self, k, d)

    c.free = Probe()
    assert c.take(2048) is None
    c.free = dict(c.free)
    assert c.take(1024) == 0x3000
