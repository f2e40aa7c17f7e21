"""Oracle transport + integrator (reference L3-L5), float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates, with identical random-number consumption so that renders are
bit-identical to the reference's on the reference's own scenes:

* SDF primitives Plane / Sphere / Box           -- sdf.py:18-84
* pinhole camera                                -- scene.py:30-51
* constant / lat-long environment               -- scene.py:61-84
* null-scattering walker (collision / ratio)    -- transport.py:70-297
* ratio-tracking transmittance estimate         -- transport.py:300-313
* wavefront integrator with sun NEE, RR         -- render.py:32-108
* tiled render with (seed, pixel) keying        -- render.py:127-180

Extensions needed by BASELINE configs that the reference lacks (recorded
conventions): grey albedo (medium.albedo), an
orthographic camera (`.ortho` cameras), and a point light (`scene.point`
with `.position` / `.intensity`, NEE weight I / r^2, shadow ray walked
in ratio mode exactly like the sun's).
"""

from __future__ import annotations

import numpy as np

from .microfacet import (density, extinction_local, kind_of, phase_eval_local,
                         phase_sample_local, projected_area, projected_area_bound, rough)
from .numerics import RayStreams, child_bases, frame_about, stream_base, to_local, to_world
from .numerics import uniform_at
from .numerics import unit, vdot


class OracleConsistencyError(RuntimeError):
    """Mirror of InternalConsistencyError (majorant excess / iteration cap)."""


# ---------------------------------------------------------------------------
# primitives (duck-typed on class name so reference and repo objects both work)


def shape_of(prim_sdf):
    return type(prim_sdf).__name__


def sdf_value(s, p):
    p = np.asarray(p, dtype=np.float64)
    k = shape_of(s)
    if k == "Plane":
        return p[..., 2] - s.z0
    if k == "Sphere":
        return np.linalg.norm(p - np.asarray(s.center), axis=-1) - s.radius
    if k == "Box":
        q = np.abs(p - np.asarray(s.center)) - np.asarray(s.half_extents)
        return np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(np.max(q, axis=-1), 0.0)
    raise TypeError(f"oracle has no SDF for {k}")


def sdf_gradient(s, p):
    p = np.asarray(p, dtype=np.float64)
    k = shape_of(s)
    if k == "Plane":
        g = np.zeros(p.shape)
        g[..., 2] = 1.0
        return g
    if k == "Sphere":
        d = p - np.asarray(s.center)
        r = np.linalg.norm(d, axis=-1, keepdims=True)
        return d / np.where(r > 0.0, r, 1.0)
    if k == "Box":
        d = p - np.asarray(s.center)
        q = np.abs(d) - np.asarray(s.half_extents)
        out = np.maximum(q, 0.0)
        on = np.linalg.norm(out, axis=-1, keepdims=True)
        g_out = np.sign(d) * out / np.where(on > 0.0, on, 1.0)
        g_in = np.eye(3)[np.argmax(q, axis=-1)] * np.where(d >= 0.0, 1.0, -1.0)
        return np.where(on > 0.0, g_out, g_in)
    raise TypeError(f"oracle has no SDF for {k}")


# Root selection for spheres.  "reference" restates transport.py:88-91
# exactly: t = t1 if t1 > 1e-12 else t2.  A ray that was just skipped onto
# the level set and whose rounded position sits a hair outside it gets
# t1 ~ 0 and is sent to the FAR root -- it tunnels through the shell (and the
# core) and escapes.  "corrected" picks the root by the side of the level
# sphere the ray is on (c = |p-c|^2 - R^2 > 0: first root, clamped >= 0;
# inside: second root), which is what the math intends.  Renders of spheres
# made with "reference" are biased; see DESIGN.md "Reference defect".
SPHERE_ROOTS = "reference"


def level_distance(s, pos, dirn, level):
    """transport.py:70-92: exact for plane/sphere (inf when unreachable),
    Lipschitz lower bound for boxes."""
    k = shape_of(s)
    if k == "Plane":
        with np.errstate(divide="ignore", invalid="ignore"):
            t = (level - sdf_value(s, pos)) / dirn[..., 2]
        return np.where(np.isfinite(t) & (t > 0.0), t, np.inf)
    if k == "Sphere":
        rad = s.radius + level
        if rad <= 0.0:
            return np.full(pos.shape[:-1], np.inf)
        oc = pos - np.asarray(s.center)
        b = vdot(oc, dirn)
        c = vdot(oc, oc) - rad * rad
        disc = b * b - c
        sq = np.sqrt(np.maximum(disc, 0.0))
        if SPHERE_ROOTS == "corrected":
            outside = c > 0.0
            t_out = np.where((b < 0.0) & (disc >= 0.0), np.maximum(-b - sq, 0.0), np.inf)
            return np.where(outside, t_out, np.maximum(-b + sq, 0.0))
        t = np.where(-b - sq > 1e-12, -b - sq, -b + sq)
        return np.where((disc >= 0.0) & (t > 1e-12), t, np.inf)
    return np.abs(sdf_value(s, pos) - level)


def slab_gap(s, pos, dirn, f, lo, hi):
    """transport.py:95-109."""
    above = f > hi
    gap = np.where(above, level_distance(s, pos, dirn, hi), level_distance(s, pos, dirn, lo))
    unreachable = np.isinf(gap)
    if shape_of(s) not in ("Plane", "Sphere"):
        unreachable = unreachable | (above & (vdot(sdf_gradient(s, pos), dirn) >= 0.0))
    return gap, unreachable


def _direction_bounds(prims, dirn):
    """transport.py:112-131: exact sigma(w) for planes, direction-free bound otherwise."""
    rows = []
    for pr in prims:
        m = pr.medium
        k = kind_of(m)
        ax, ay, az = rough(m)
        if shape_of(pr.sdf) == "Plane":
            rows.append(np.broadcast_to(np.asarray(projected_area(dirn, k, ax, ay, az)),
                                        dirn.shape[:-1]))
        else:
            rows.append(np.full(dirn.shape[:-1], projected_area_bound(k, ax, ay, az)))
    return np.stack(rows, axis=0)


# ---------------------------------------------------------------------------
# walker (transport.py:144-297)

MAX_WALK_STEPS = 200000


def walk(prims, pos, dirn, streams, ratio_mode=False):
    """Advance every ray to escape (0), absorption (1) or a real collision (2).

    Returns (state, pos, travel, weight, prim).  Streams advance in place."""
    n = np.asarray(pos).shape[0]
    st_out = np.zeros(n, dtype=np.int8)
    p_out = np.array(pos, dtype=np.float64)
    t_out = np.zeros(n)
    w_out = np.ones(n)
    k_out = np.full(n, -1, dtype=np.int64)
    if not prims:
        return st_out, p_out, t_out, w_out, k_out
    sig = np.array([pr.medium.sigma for pr in prims])
    half = 0.5 * sig
    lo = (-3.0 if ratio_mode else -6.0) * sig
    hi = 3.0 * sig
    min_skip = 1e-7 * float(np.min(sig))
    n_p = len(prims)

    live = np.arange(n)
    p = p_out.copy()
    d = np.array(dirn, dtype=np.float64)
    trav = np.zeros(n)
    wgt = np.ones(n)
    base = np.array(np.broadcast_to(streams.base, (n,)), dtype=np.uint64)
    ctr = np.array(np.broadcast_to(streams.counter, (n,)), dtype=np.uint64)
    bound = _direction_bounds(prims, d)

    def finish(rows, code):
        g = live[rows]
        st_out[g] = code
        p_out[g] = p[g]
        t_out[g] = trav[g]
        w_out[g] = wgt[g]

    for _ in range(MAX_WALK_STEPS):
        if live.size == 0:
            streams.counter = ctr
            return st_out, p_out, t_out, w_out, k_out
        pl = p[live]
        dl = d[live]
        f = np.stack([np.asarray(sdf_value(pr.sdf, pl)) for pr in prims], axis=0)
        gone = np.zeros(live.size, dtype=bool)
        if not ratio_mode:
            deep = np.any(f < lo[:, None], axis=0)
            finish(np.flatnonzero(deep), 1)
            gone |= deep
        band = (f >= lo[:, None]) & (f <= hi[:, None])
        gaps = np.empty((n_p, live.size))
        fin = np.empty((n_p, live.size), dtype=bool)
        for j, pr in enumerate(prims):
            g, u = slab_gap(pr.sdf, pl, dl, f[j], lo[j], hi[j])
            gaps[j] = np.where(band[j], np.inf, g)
            fin[j] = ~band[j] & u
        inside_any = np.any(band, axis=0)

        vac = ~inside_any & ~gone
        esc = vac & np.all(fin, axis=0)
        finish(np.flatnonzero(esc), 0)
        gone |= esc
        mv = vac & ~gone
        if np.any(mv):
            jump = np.maximum(np.min(gaps, axis=0), min_skip)
            rows = live[mv]
            p[rows] += d[rows] * jump[mv][:, None]
            trav[rows] += jump[mv]

        stp = inside_any & ~gone
        if np.any(stp):
            bnd = band & stp[None, :]
            maj = np.zeros(live.size)
            for j in range(n_p):
                fb = np.maximum(f[j] - half[j], lo[j])
                maj += np.where(bnd[j], density(fb, sig[j]) * bound[j, live], 0.0)
            cap = np.min(np.where(bnd, half[:, None], np.maximum(gaps, min_skip)), axis=0)
            u1 = uniform_at(base[live], ctr[live])
            ctr[live] += stp.astype(np.uint64)
            with np.errstate(divide="ignore", invalid="ignore"):
                dt = np.where(maj > 0.0, -np.log1p(-u1) / maj, np.inf)
            hit = stp & (dt <= cap)
            adv = np.where(stp, np.where(hit, dt, cap), 0.0)
            p[live] += dl * adv[:, None]
            trav[live] += adv

            hr = np.flatnonzero(hit)
            if hr.size:
                gl = live[hr]
                ph = p[gl]
                dh = d[gl]
                parts = np.zeros((n_p, hr.size))
                for j, pr in enumerate(prims):
                    fc = np.asarray(sdf_value(pr.sdf, ph))
                    ins = (fc >= lo[j]) & (fc <= hi[j])
                    if not np.any(ins):
                        continue
                    wl = to_local(frame_about(sdf_gradient(pr.sdf, ph)), dh)
                    sj = extinction_local(wl, np.where(ins, fc, 0.0), pr.medium)
                    parts[j] = np.where(ins, sj, 0.0)
                tot = np.sum(parts, axis=0)
                ratio = tot / maj[hr]
                if np.any(ratio > 1.0 + 1e-9):
                    raise OracleConsistencyError(
                        f"extinction exceeded its majorant (ratio {float(np.max(ratio)):.6g})")
                if ratio_mode:
                    wgt[gl] *= np.maximum(1.0 - ratio, 0.0)
                else:
                    u2 = uniform_at(base[gl], ctr[gl])
                    ctr[gl] += np.uint64(1)
                    real = u2 < ratio
                    if np.any(real):
                        cum = np.cumsum(parts, axis=0)
                        choice = np.argmax(cum > (u2 * maj[hr])[None, :], axis=0)
                        k_out[gl[real]] = choice[real]
                        finish(hr[real], 2)
                        gone[hr[real]] = True
        live = live[~gone]
    raise OracleConsistencyError("walker exceeded its iteration cap")


def transmittance_estimate(origin, direction, prims, n, seed, stream):
    """transport.py:300-313: mean and standard error of ratio tracking."""
    n = int(n)
    rs = RayStreams(child_bases(seed, stream, np.arange(n)), np.zeros(n, dtype=np.uint64))
    pos = np.broadcast_to(np.asarray(origin, dtype=np.float64), (n, 3))
    dirs = np.broadcast_to(np.asarray(direction, dtype=np.float64), (n, 3))
    state, _, _, w, _ = walk(prims, pos, dirs, rs, ratio_mode=True)
    w = np.where(state == 1, 0.0, w)
    se = float(np.std(w, ddof=1) / np.sqrt(n)) if n > 1 else 0.0
    return float(np.mean(w)), se


# ---------------------------------------------------------------------------
# cameras, environment


def camera_basis(cam):
    """scene.py:30-41 basis (forward, right, true-up)."""
    pos = np.asarray(cam.position, dtype=np.float64)
    fwd = unit(np.asarray(cam.look_at, dtype=np.float64) - pos)
    up = np.array([0.0, 0.0, 1.0])
    if abs(fwd @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = unit(np.cross(fwd, up))
    return pos, fwd, right, np.cross(right, fwd)


def camera_rays(cam, px, py, jx, jy):
    """Pinhole (scene.py:30-51) or, for cameras with `.ortho` true, the
    orthographic extension: film of `.film_height` world units centred on
    `.position`, rays parallel to the view axis."""
    pos, fwd, right, tup = camera_basis(cam)
    nx = ((px + jx) / cam.width) * 2.0 - 1.0
    ny = 1.0 - ((py + jy) / cam.height) * 2.0
    if getattr(cam, "ortho", False):
        hh = 0.5 * cam.film_height
        hw = hh * cam.width / cam.height
        o = pos + nx[..., None] * hw * right + ny[..., None] * hh * tup
        return o, np.broadcast_to(fwd, o.shape).copy()
    hh = np.tan(0.5 * np.deg2rad(cam.fov_deg))
    hw = hh * cam.width / cam.height
    d = unit(fwd + nx[..., None] * hw * right + ny[..., None] * hh * tup)
    return np.broadcast_to(pos, d.shape).copy(), d


def env_radiance(env, d):
    """scene.py:61-84."""
    d = np.asarray(d, dtype=np.float64)
    img = getattr(env, "latlong", None)
    if img is None:
        return np.broadcast_to(np.asarray(env.radiance, dtype=np.float64), d.shape[:-1] + (3,))
    h, w = img.shape[:2]
    th = np.arccos(np.clip(d[..., 2], -1.0, 1.0))
    ph = np.mod(np.arctan2(d[..., 1], d[..., 0]), 2.0 * np.pi)
    fx = ph / (2.0 * np.pi) * w - 0.5
    fy = th / np.pi * h - 0.5
    x0 = np.floor(fx).astype(int)
    y0 = np.floor(fy).astype(int)
    tx = (fx - x0)[..., None]
    ty = (fy - y0)[..., None]
    xa, xb = x0 % w, (x0 + 1) % w
    ya, yb = np.clip(y0, 0, h - 1), np.clip(y0 + 1, 0, h - 1)
    return (img[ya, xa] * (1 - tx) * (1 - ty) + img[ya, xb] * tx * (1 - ty)
            + img[yb, xa] * (1 - tx) * ty + img[yb, xb] * tx * ty)


# ---------------------------------------------------------------------------
# integrator (render.py:32-108)

RR_AFTER = 8            # render.py:27
SEGMENT_CAP = 4096      # render.py:29
SAMPLE_STRIDE = np.uint64(1) << np.uint64(28)   # render.py:28


def _nee(scene, prims, rows, pos, dirs, throughput, radiance, streams, j):
    """Sun NEE (render.py:71-82) and the repo's point-light extension."""
    med = prims[j].medium
    frame = frame_about(sdf_gradient(prims[j].sdf, pos[rows]))
    wo_l = to_local(frame, dirs[rows])
    lights = []
    sun = getattr(scene, "sun", None)
    if sun is not None:
        wl = np.broadcast_to(-np.asarray(sun.direction, dtype=np.float64), (rows.size, 3))
        lights.append((wl, np.asarray(sun.radiance, dtype=np.float64)[None, :]))
    pt = getattr(scene, "point", None)
    if pt is not None:
        to = np.asarray(pt.position, dtype=np.float64) - pos[rows]
        r2 = vdot(to, to)
        wl = to / np.sqrt(r2)[:, None]
        lights.append((wl, np.asarray(pt.intensity, dtype=np.float64)[None, :] / r2[:, None]))
    for wl, le in lights:
        ph = phase_eval_local(wo_l, to_local(frame, wl), med)
        sub = streams.subset(rows)
        s_state, _, _, s_w, _ = walk(prims, pos[rows], np.array(wl), sub, ratio_mode=True)
        streams.merge(rows, sub)
        tr = np.where(s_state == 1, 0.0, s_w)
        radiance[rows] += throughput[rows] * ph * tr[:, None] * le
    return frame, wo_l


def trace_paths(origins, directions, scene, max_bounces, streams):
    """Trace a wavefront of paths to completion; returns (N, 3) radiance."""
    if max_bounces < 1:
        raise ValueError(f"max_bounces must be >= 1, got {max_bounces}")
    prims = tuple(scene.primitives)
    pos = np.array(origins, dtype=np.float64)
    dirs = np.array(directions, dtype=np.float64)
    n = pos.shape[0]
    L = np.zeros((n, 3))
    T = np.ones((n, 3))
    alive = np.ones(n, dtype=bool)
    depth = np.zeros(n, dtype=np.int64)
    for _ in range(SEGMENT_CAP):
        idx = np.flatnonzero(alive)
        if idx.size == 0:
            break
        sub = streams.subset(idx)
        state, p_end, _, _, pk = walk(prims, pos[idx], dirs[idx], sub)
        streams.merge(idx, sub)
        pos[idx] = p_end
        esc = idx[state == 0]
        if esc.size:
            L[esc] += T[esc] * env_radiance(scene.environment, dirs[esc])
            alive[esc] = False
        alive[idx[state == 1]] = False
        hit = idx[state == 2]
        if hit.size == 0:
            continue
        which = pk[state == 2]
        for j in range(len(prims)):
            rows = hit[which == j]
            if rows.size == 0:
                continue
            frame, wo_l = _nee(scene, prims, rows, pos, dirs, T, L, streams, j)
            sub = streams.subset(rows)
            u = np.stack([sub.draw(), sub.draw(), sub.draw()], axis=-1)
            streams.merge(rows, sub)
            wi_l, _, wt = phase_sample_local(wo_l, prims[j].medium, u)
            dirs[rows] = to_world(frame, wi_l)
            T[rows] *= wt
        depth[hit] += 1
        alive[hit[depth[hit] >= max_bounces]] = False
        rr = hit[(depth[hit] > RR_AFTER) & alive[hit]]
        if rr.size:
            q = np.minimum(np.max(T[rr], axis=1), 1.0)
            sub = streams.subset(rr)
            u = sub.draw()
            streams.merge(rr, sub)
            die = u >= q
            alive[rr[die]] = False
            T[rr[~die]] /= q[~die][:, None]
    return L


def render_tile(scene, spp, seed, max_bounces, ys, xs, tile=32):
    """One tile of render.py:141-166; returns (ye, xe, (h, w, 3) mean radiance)."""
    cam = scene.camera
    w, h = cam.width, cam.height
    ye, xe = min(h, ys + tile), min(w, xs + tile)
    yy, xx = np.mgrid[ys:ye, xs:xe]
    pix = (yy * w + xx).ravel()
    npx = pix.size
    base = stream_base(np.uint64(seed), pix.astype(np.uint64))
    acc = np.zeros((npx, 3))
    block = max(1, min(spp, 131072 // max(1, tile * tile)))
    for s0 in range(0, spp, block):
        ns = min(block, spp - s0)
        rs = RayStreams(np.repeat(base, ns),
                        np.tile(np.arange(s0, s0 + ns, dtype=np.uint64), npx) * SAMPLE_STRIDE)
        jx = rs.draw()
        jy = rs.draw()
        o, d = camera_rays(cam, np.repeat(xx.ravel(), ns), np.repeat(yy.ravel(), ns), jx, jy)
        acc += trace_paths(o, d, scene, max_bounces, rs).reshape(npx, ns, 3).sum(axis=1)
    return ye, xe, (acc / spp).reshape(ye - ys, xe - xs, 3)


def render(scene, spp, seed, max_bounces=64, tile=32):
    """render.py:127-180 (serial); returns the (H, W, 3) float64 image."""
    cam = scene.camera
    out = np.zeros((cam.height, cam.width, 3))
    for ys in range(0, cam.height, tile):
        for xs in range(0, cam.width, tile):
            ye, xe, img = render_tile(scene, spp, seed, max_bounces, ys, xs, tile)
            out[ys:ye, xs:xe] = img
    return out
