"""CPU timing harness for the oracle port -- TEST / BENCH INFRASTRUCTURE ONLY.

Reproduces the reference render()'s work decomposition (render.py:127-174:
32x32 tiles, sample blocks of <= 131072 paths, RNG keyed by (seed, pixel)
with counter block s * 2^28) through `oracle.tracer.render_tile`, fanned
out over a process pool -- the reference's own thread pool is GIL-bound
(SURVEY.md section 6), so processes are the fair CPU baseline.
Used by bench.py's `cpu_baseline` leg and `--impl reference` arm only.

A pool serves a LIST of scenes (the nine config-4 panels); every job names
its scene, so one timed step can cover a workload mix with the same number
of paths per scene as the GPU step.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

_SCENES = None


def _init(scenes):
    global _SCENES
    _SCENES = scenes
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"


def _job(args):
    from .tracer import render_tile

    k, spp, seed, max_bounces, ys, xs, tile = args
    ye, xe, img = render_tile(_SCENES[k], spp, seed, max_bounces, ys, xs, tile)
    return (ye - ys) * (xe - xs) * spp, float(img.sum())


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _tiles(scene, tile):
    cam = scene.camera
    return [(ys, xs) for ys in range(0, cam.height, tile) for xs in range(0, cam.width, tile)]


def run_jobs(jobs, pool=None, scenes=None):
    """Run (scene index, spp, seed, depth, ys, xs, tile) jobs; returns
    (paths, seconds)."""
    t0 = time.perf_counter()
    if pool is not None:
        res = pool.map(_job, jobs, chunksize=1)
    else:
        _init(scenes)
        res = [_job(j) for j in jobs]
    dt = time.perf_counter() - t0
    return sum(r[0] for r in res), dt


def make_pool(scenes, workers):
    ctx = mp.get_context("fork")
    return ctx.Pool(processes=workers, initializer=_init, initargs=(list(scenes),))


def mix_jobs(scenes, seed, max_bounces, paths_per_scene, jobs_per_scene, tile=32):
    """Equal paths per scene, each scene's share split into jobs_per_scene
    tile jobs (distinct tiles, the reference's wavefront size at most)."""
    jobs = []
    for k, sc in enumerate(scenes):
        tiles = _tiles(sc, tile)
        per_job = max(1, paths_per_scene // jobs_per_scene)
        spp = max(1, round(per_job / (tile * tile)))
        for j in range(jobs_per_scene):
            ys, xs = tiles[(j * 7919) % len(tiles)]
            jobs.append((k, spp, seed, max_bounces, ys, xs, tile))
    return jobs


def calibrated_mix(scenes, seed, max_bounces, budget_s, workers, tile=32):
    """Jobs for one step of about budget_s on `workers` processes with
    equal paths per scene: the single-core rate of every scene is measured
    on a small tile job first."""
    secs_per_path = 0.0
    for k in range(len(scenes)):
        p, dt = run_jobs([(k, 4, seed, max_bounces, 0, 0, tile)], scenes=scenes)
        secs_per_path += dt / p
    secs_per_path /= len(scenes)                   # mean single-core cost
    total = workers * budget_s / secs_per_path     # paths in the budget
    per_scene = int(max(tile * tile, total / len(scenes)))
    jobs_per_scene = max(1, -(-2 * workers // len(scenes)))
    return mix_jobs(scenes, seed, max_bounces, per_scene, jobs_per_scene, tile), 1.0 / secs_per_path


def describe(jobs, scenes_label, workers):
    paths = sum(j[1] * j[6] * j[6] for j in jobs)
    return (f"{len(jobs)} tile jobs ({jobs[0][6]}x{jobs[0][6]} px, spp {jobs[0][1]}) over "
            f"{scenes_label}, {paths} paths, oracle/tracer.py (float64 numpy restatement of the "
            f"reference walk/trace_paths/render_tile, identical RNG consumption) on {workers} "
            "processes")
