"""Frozen algorithmic work counts for the FP32 / SFU issue roofline.

SURVEY.md 8(d): the per-unit work is counted from the fp32 SOURCE FORMULAS
of csrc/mf_math.cuh / mf_transport.cuh (not from SASS), per device event,
and multiplied by the event counters the kernels report (mf_stats):

    F = sum_e count_e * fp32_e      (FMA / FMUL / FADD, integer IMAD of
                                     Philox; 1 each on the FMA pipe)
    S = sum_e count_e * sfu_e       (MUFU RCP / RSQ / SQRT / EX2 / LG2)
    roofline fraction = max(F / P_fp32, S / P_sfu) / T_kernel

Comparisons, selects, min/max, integer logic and conversions are NOT
counted (ALU pipe); neither are divergence and re-convergence.  The
peaks P are measured on the device by mf_measure_peaks (FFMA / MUFU.EX2
microbenchmarks).  The per-primitive costs below are the counts of the
formulas as written (library expf = 3 F + 1 S, logf = 10 F, log1pf = 12
F, approximate division / sqrt = 1 F + 1 S).
"""

from __future__ import annotations

# cost of the building blocks, (fp32, sfu)
PRIMS = {
    "erfcx": (16, 1),
    "ierfcx": (18, 1),
    "erfcx_pair": (32, 1),
    "exp_neg_sq": (7, 1),
    "mills": (22, 2.5),
    "log_ndtr": (35, 1.5),
    "ndtri": (27, 0),
    "inv_log_ndtr": (89, 5),
    "proj_area": (33, 3),
    "frame": (10, 1),
    "rotate": (9, 0),
    "ndf_generalized": (45, 4.5),
    "ndf_beckmann": (10, 2),
    "phase_eval": (67, 8.5),
    "mixture_pdf": (16, 3),
    "philox": (44, 0),
    "slope_log_cdf": (52, 2.5),
}

# per-event costs, (fp32, sfu)
EVENTS = {
    # raygen: Philox block + orthographic / pinhole camera ray
    "paths": (54, 2),
    # free-flight segment: Philox block + sigma(dir) + analytic planar flight
    # (log(u), log_ndtr, division, inv_log_ndtr, position update)
    "segments": (212, 12.5),
    # real scatter: frame + sigma(wo) + phase sample (sigma_b, branch remap,
    # mixture pdf, vNDF weight, 50/50 Beckmann (55 + 110 base + one residual
    # evaluation 57 from the table guess) / hemisphere (43) proposal,
    # rotation, throughput, RR)
    "scatters": (304, 28),
    # next-event estimation: phase_eval + sigma(wl) + closed-form / walk Tr
    "nee": (157, 15),
    # each further Newton iteration of the visible-slope inversion
    "slope_iters": (57, 3.5),
    # one delta / ratio tracking step on a curved shell (majorant, sample,
    # tentative extinction)
    "track_steps": (70, 8),
}


# Single-plane scenes without a point light (configs 2, 4; pool_kernel):
#   - the flight is sampled in log-Phi space from the previous collision's
#     carried log Phi: Philox block + 4 uniforms + sigma(dir) + log(u) + the
#     log-Phi step (no log_ndtr, and no inv_log_ndtr since no position is
#     read; an entry from above starts at the constant log Phi(3));
#   - the scatter reuses sigma(dir) as sigma(wo) (identity frame);
#   - NEE to the sun: phase_eval + the closed-form transmittance from the
#     carried log Phi (clamp, one exp), sigma(w_sun) precomputed per render.
PLANAR_EVENTS = {
    "paths": EVENTS["paths"],
    "segments": (44 + 4 + PRIMS["proj_area"][0] + 1 + 2 + 1, PRIMS["proj_area"][1] + 3),
    "scatters": (EVENTS["scatters"][0] - PRIMS["proj_area"][0],
                 EVENTS["scatters"][1] - PRIMS["proj_area"][1]),
    "nee": (9 + PRIMS["phase_eval"][0] + 5 + 3 + 9, PRIMS["phase_eval"][1] + 2),
    "slope_iters": EVENTS["slope_iters"],
    "track_steps": EVENTS["track_steps"],
}


# One config-1 coefficient query (query_kernel): the scatter event's phase
# sample (sigma_b, branch remap, 50/50 Beckmann / hemisphere proposal,
# mixture pdf, vNDF weight, frame and rotations) + phase_eval of wi + the
# density of sigma_t (mills and 3 multiplies) + the pdf of wi (half vector,
# mixture pdf) + the two rotations of wo, wi into the local frame.
QUERY = (EVENTS["scatters"][0] + PRIMS["phase_eval"][0] + PRIMS["mills"][0] + 3
         + 9 + PRIMS["mixture_pdf"][0] + 3 + 2 * PRIMS["rotate"][0],
         EVENTS["scatters"][1] + PRIMS["phase_eval"][1] + PRIMS["mills"][1]
         + 1 + PRIMS["mixture_pdf"][1])


def query_roofline(n_queries, kernel_ms, peak_fp32_ginst, peak_sfu_ginst):
    """Roofline fraction of the query kernel from the per-query count QUERY."""
    t = kernel_ms * 1e-3
    af = n_queries * QUERY[0] / t / 1e9
    asf = n_queries * QUERY[1] / t / 1e9
    ff, fs = af / peak_fp32_ginst, asf / peak_sfu_ginst
    return {"bound": "fp32" if ff >= fs else "sfu", "frac": max(ff, fs), "fp32_frac": ff,
            "sfu_frac": fs, "fp32_per_query": QUERY[0], "sfu_per_query": QUERY[1]}


# bytes one config-1 query moves: 11 float32 inputs + 13 outputs (sigma_t,
# phase rgb, pdf, sampled direction, pdf_s, weight rgb, flags)
QUERY_BYTES = 11 * 4 + 13 * 4

# Beckmann media (config-4 panels with l_z = inf) evaluate the height-field
# NDF instead of the generalized one in phase_eval (NEE) and in the sample
# weight (scatter): the difference of the two NDF costs per such event
_BECK_DIFF = (PRIMS["ndf_generalized"][0] - PRIMS["ndf_beckmann"][0],
              PRIMS["ndf_generalized"][1] - PRIMS["ndf_beckmann"][1])


def algorithmic_ops(stats, planar=False, kind=None):
    """(fp32 lane ops, sfu lane ops) of a render from its mf_stats counters;
    planar=True: the sun-lit single-plane event costs (PLANAR_EVENTS);
    kind: the medium's NdfKind (BECKMANN media count the cheaper NDF)."""
    f = s = 0.0
    for ev, (cf, cs) in (PLANAR_EVENTS if planar else EVENTS).items():
        n = float(stats.get(ev, 0))
        f += n * cf
        s += n * cs
    if kind is not None and getattr(kind, "value", kind) == "beckmann":
        n = float(stats.get("nee", 0)) + float(stats.get("scatters", 0))
        f -= n * _BECK_DIFF[0]
        s -= n * _BECK_DIFF[1]
    return f, s


def from_ops(f, s, kernel_ms, peak_fp32_ginst, peak_sfu_ginst, paths=1):
    """Achieved issue rates and the roofline fraction for f / s algorithmic
    lane ops executed in kernel_ms."""
    t = kernel_ms * 1e-3
    af = f / t / 1e9
    asf = s / t / 1e9
    ff = af / peak_fp32_ginst
    fs = asf / peak_sfu_ginst
    bound = "fp32" if ff >= fs else "sfu"
    return {
        "bound": bound,
        "achieved": af if bound == "fp32" else asf,
        "peak": peak_fp32_ginst if bound == "fp32" else peak_sfu_ginst,
        "unit": "Ginst/s",
        "frac": max(ff, fs),
        "fp32_frac": ff,
        "sfu_frac": fs,
        "fp32_per_path": f / max(float(paths), 1.0),
        "sfu_per_path": s / max(float(paths), 1.0),
    }


def roofline(stats, kernel_ms, peak_fp32_ginst, peak_sfu_ginst, planar=False, kind=None):
    """Achieved issue rates and the roofline fraction of the path kernel."""
    f, s = algorithmic_ops(stats, planar, kind)
    return from_ops(f, s, kernel_ms, peak_fp32_ginst, peak_sfu_ginst, stats.get("paths", 1))
