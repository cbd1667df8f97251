"""Comparison statistics shared by the Eigen-association parity tests (test
infrastructure): two volumes / map pairs -> the §8(c) tolerance measures."""
from __future__ import annotations

import numpy as np

from helpers import allocated_blocks


def positions(entries):
    e = entries[entries["block_state"] >= 0]
    return set(zip(e["x"].tolist(), e["y"].tolist(), e["z"].tolist()))


def compare(ea, va, eb, vb, maps_a, maps_b, voxel_size):
    sa, sb = positions(ea), positions(eb)
    ba, bb = allocated_blocks(ea, va, 4), allocated_blocks(eb, vb, 4)
    keys = sorted(set(ba) & set(bb))
    sdf_a = np.stack([ba[k][:, :2].copy().view(np.int16)[:, 0] for k in keys]).astype(np.int64)
    sdf_b = np.stack([bb[k][:, :2].copy().view(np.int16)[:, 0] for k in keys]).astype(np.int64)
    w_a = np.stack([ba[k][:, 2] for k in keys]).astype(np.int64)
    w_b = np.stack([bb[k][:, 2] for k in keys]).astype(np.int64)
    d = np.abs(sdf_a - sdf_b)
    (pa, na), (pb, nb) = maps_a, maps_b
    ha, hb = pa[..., 3] > 0, pb[..., 3] > 0
    both = ha & hb
    dp = np.linalg.norm(pa[..., :3] - pb[..., :3], axis=-1)[both]
    cos = np.clip((na[..., :3] * nb[..., :3]).sum(-1)[both], -1.0, 1.0)
    ang = np.degrees(np.arccos(cos))
    return {
        "blocks": [len(sa), len(sb)], "blocks_common_frac": len(sa & sb) / max(len(sa), len(sb), 1),
        "sdf_exact_frac": float(np.mean(d == 0)), "sdf_le1_frac": float(np.mean(d <= 1)),
        "sdf_le64_frac": float(np.mean(d <= 64)), "weight_exact_frac": float(np.mean(w_a == w_b)),
        "maps_bit_exact_frac": float(np.mean((pa.view(np.uint32) == pb.view(np.uint32)).all(-1))),
        "hit_agreement": float(np.mean(ha == hb)),
        "point_within_half_voxel_frac": float(np.mean(dp <= 0.5 * voxel_size)),
        "point_max_m": float(dp.max()) if dp.size else 0.0,
        "normal_within_1deg_frac": float(np.mean(ang <= 1.0)),
        "normal_max_deg": float(ang.max()) if ang.size else 0.0,
    }
