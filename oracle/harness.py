"""CPU timing harness for the oracle port -- TEST / BENCH INFRASTRUCTURE ONLY.

Reproduces the reference render()'s work decomposition (render.py:127-174:
32x32 tiles, sample blocks of <= 131072 paths, RNG keyed by (seed, pixel)
with counter block s * 2^28) through `oracle.tracer.render_tile`, fanned
out over a process pool -- the reference's own thread pool is GIL-bound
(SURVEY.md section 6), so processes are the fair CPU baseline.
Used by bench.py's `cpu_baseline` leg and `--impl reference` arm only.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

_SCENE = None


def _init(scene):
    global _SCENE
    _SCENE = scene
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"


def _job(args):
    from .tracer import render_tile

    spp, seed, max_bounces, ys, xs, tile = args
    ye, xe, img = render_tile(_SCENE, spp, seed, max_bounces, ys, xs, tile)
    return (ye - ys) * (xe - xs) * spp, float(img.sum())


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def tile_jobs(scene, spp, seed, max_bounces, n_tiles, tile=32):
    cam = scene.camera
    jobs = []
    for ys in range(0, cam.height, tile):
        for xs in range(0, cam.width, tile):
            jobs.append((spp, seed, max_bounces, ys, xs, tile))
    return jobs[:n_tiles]


def timed_render(scene, spp, seed, max_bounces, n_tiles, workers, tile=32, pool=None):
    """Render the first n_tiles tiles at `spp`; returns (paths, seconds)."""
    jobs = tile_jobs(scene, spp, seed, max_bounces, n_tiles, tile)
    t0 = time.perf_counter()
    if pool is not None:
        res = pool.map(_job, jobs, chunksize=1)
    else:
        _init(scene)
        res = [_job(j) for j in jobs]
    dt = time.perf_counter() - t0
    return sum(r[0] for r in res), dt


def make_pool(scene, workers):
    ctx = mp.get_context("fork")
    return ctx.Pool(processes=workers, initializer=_init, initargs=(scene,))


def calibrated_sample(scene, max_bounces, seed, budget_s, workers, tile=32, pool=None):
    """Pick (spp, n_tiles) so one timed_render takes about budget_s on
    `workers` processes.  Per-tile jobs use the reference's own wavefront
    size (render.py:141-142: 131072 paths = 128 spp of a 32x32 tile), so
    numpy batching is as efficient as in the reference's render()."""
    per_tile = tile * tile
    spp = max(1, 131072 // per_tile)
    paths, dt = timed_render(scene, max(1, spp // 4), seed, max_bounces, 1, 1, tile)
    rate1 = paths / max(dt, 1e-6)           # paths/s on one core
    target = rate1 * workers * budget_s      # paths in the budget
    n_img = ((scene.camera.height + tile - 1) // tile) * ((scene.camera.width + tile - 1) // tile)
    n_tiles = int(max(1, min(n_img, round(target / (spp * per_tile)))))
    if n_tiles < workers:
        # fewer jobs than cores: keep every core busy with smaller sample blocks
        n_tiles = min(n_img, workers)
        spp = max(1, int(target / (n_tiles * per_tile)))
    return spp, n_tiles, rate1
