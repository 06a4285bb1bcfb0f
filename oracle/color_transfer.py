"""CPU restatement of colour transfer — TEST INFRASTRUCTURE ONLY.

Follows /root/reference/proj/include/pot/color_transfer.hpp:
  kmeans_quantize          :34-118  (C++ oracle: binding.kmeans)
  barycentric_projection   :128-141
  color_transfer           :146-185 (the solve in the C++ oracle)
Pinned by the reference's Kmeans*, Barycentric*, ColorTransfer* tests
(test_apps.cpp:38-160), ported in tests/test_oracle_color.py.
"""
from __future__ import annotations

import numpy as np

from . import binding


def barycentric_projection(plan, source, target):
    out = np.array(source, dtype=np.float64, copy=True)
    for i in range(plan.shape[0]):
        m = plan[i].sum()
        if m > 0:
            out[i] = (plan[i] @ target) / m
    return out


def color_transfer(src_c, src_w, tgt_c, tgt_w, s_frac, kind, epsilon=0.1, p=1.0, max_iterations=50000):
    norm = max(src_w.sum(), tgt_w.sum())
    r, c = src_w / norm, tgt_w / norm
    d = src_c[:, None, :] - tgt_c[None, :, :]
    C = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
    cmax = C.max()
    if cmax > 0:
        C = C / cmax
    s = s_frac * min(r.sum(), c.sum())
    res = binding.solve(kind, r, c, s, C=C, epsilon=epsilon, p=p, max_iterations=max_iterations)
    return barycentric_projection(res.plan, src_c, tgt_c), res, (r, c, C, s)
