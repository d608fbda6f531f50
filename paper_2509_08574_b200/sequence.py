"""Repeated-scan driver (BASELINE config c5).

A prior image, then a sequence of sparse follow-up scans, each reconstructed
with IRN-PICCS warm-started from the previous follow-up's result through
``ReconOptions.initial`` (recon.hpp:68-72, :157) — so τ is resolved from the
initial image (recon.hpp:161-162), exactly as a chain of reference calls
``irn_piccs(proj_t, grid, prior, params, {.initial = &x_{t-1}})`` would.
Everything stays on the device when the inputs are CUDA tensors.
"""
from __future__ import annotations

import time

from . import ConeBeamProjector, ProjectionSet, ReconOptions, irn_piccs


def repeated_scan(projector: ConeBeamProjector, followups, prior, params, initial=None,
                  ground_truths=None, layout=None):
    """Reconstruct each follow-up in turn; returns (reports, seconds per follow-up).

    followups: sequence of projection arrays (one per follow-up scan, all on the
    projector's geometry); prior: the prior image; initial: start of the first
    follow-up (None = zeros, like the reference)."""
    x = initial
    reports, seconds = [], []
    for t, b in enumerate(followups):
        opts = ReconOptions(initial=x,
                            ground_truth=None if ground_truths is None else ground_truths[t])
        t0 = time.perf_counter()
        rep = irn_piccs(ProjectionSet(projector.geometry, b), projector.grid, prior, params, opts,
                        projector=projector, layout=layout)
        seconds.append(time.perf_counter() - t0)
        reports.append(rep)
        x = rep.volume
    return reports, seconds
