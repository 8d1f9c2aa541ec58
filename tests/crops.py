"""Lateral crops of BASELINE-size workloads for sampled full-size parity (tests only).

A crop keeps the full depth, N, h, materials, interface, plane wave and every PMUT overlapping the
window (windows are aligned so no membrane is cut); faces of the window that are not faces of the
full box become rigid.  After k steps, a node's value is exact in the crop if every element and
interface face that the k-step dependency cone of that node touches lies inside the crop; for the
2-step comparisons used here a margin of one coarse element (two fine) suffices.
"""
import numpy as np

from sem_inputs import BC_RIGID


def crop_record(rec, win, margin_fine=2):
    """win = (ex0, ex1, ey0, ey1) in box-0 element units.  Returns (crop_rec, info)."""
    full_boxes = rec["boxes"]
    R = 1
    if len(full_boxes) == 2:
        R = full_boxes[0]["nel"][0] // full_boxes[1]["nel"][0]
        assert all(w % R == 0 for w in win), "window must be coarse-aligned"
    boxes, info = [], {"maps": [], "valid": []}
    for bi, b in enumerate(full_boxes):
        s = 1 if bi == 0 else R
        ex0, ex1, ey0, ey1 = win[0] // s, win[1] // s, win[2] // s, win[3] // s
        h = [b["extent"][d] / b["nel"][d] for d in range(3)]
        nb = dict(b)
        nb["origin"] = (b["origin"][0] + h[0] * ex0, b["origin"][1] + h[1] * ey0, b["origin"][2])
        nb["extent"] = (h[0] * (ex1 - ex0), h[1] * (ey1 - ey0), b["extent"][2])
        nb["nel"] = (ex1 - ex0, ey1 - ey0, b["nel"][2])
        bc = list(b["bc"])
        real = [ex0 == 0, ex1 == b["nel"][0], ey0 == 0, ey1 == b["nel"][1]]
        for f in range(4):
            if not real[f]:
                bc[f] = BC_RIGID
        nb["bc"] = bc
        boxes.append(nb)
        N = b["degree"]
        NXf, NYf = N * b["nel"][0] + 1, N * b["nel"][1] + 1
        nx, ny, nz = N * (ex1 - ex0) + 1, N * (ey1 - ey0) + 1, N * b["nel"][2] + 1
        gz, gy, gx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        gx, gy, gz = gx.ravel(), gy.ravel(), gz.ravel()
        full = (gx + N * ex0) + NXf * ((gy + N * ey0) + NYf * gz)
        m = max(1, -(-margin_fine // s)) * N           # margin in lattice points
        ok = np.ones(gx.shape, bool)
        if not real[0]:
            ok &= gx >= m
        if not real[1]:
            ok &= gx <= nx - 1 - m
        if not real[2]:
            ok &= gy >= m
        if not real[3]:
            ok &= gy <= ny - 1 - m
        info["maps"].append(full.astype(np.int64))
        info["valid"].append(ok)
    crop = dict(rec)
    crop["boxes"] = boxes
    crop["name"] = rec["name"] + f"_crop{win}"
    pm = rec.get("pmut")
    info["pmut_full_index"] = []
    info["pmut_valid"] = []
    if pm is not None:
        b0 = full_boxes[0]
        h0 = b0["extent"][0] / b0["nel"][0]
        x0, x1 = b0["origin"][0] + h0 * win[0], b0["origin"][0] + h0 * win[1]
        y0, y1 = b0["origin"][1] + h0 * win[2], b0["origin"][1] + h0 * win[3]
        a = pm["side"]
        keep = []
        for k, (cx, cy) in enumerate(pm["centers"]):
            lo_x, hi_x, lo_y, hi_y = cx - a / 2, cx + a / 2, cy - a / 2, cy + a / 2
            overlap = hi_x > x0 and lo_x < x1 and hi_y > y0 and lo_y < y1
            if not overlap:
                continue
            assert lo_x >= x0 and hi_x <= x1 and lo_y >= y0 and hi_y <= y1, "window cuts a membrane"
            keep.append(k)
            mm = margin_fine * h0
            valid = ((lo_x - x0 >= mm or win[0] == 0) and (x1 - hi_x >= mm or win[1] == b0["nel"][0])
                     and (lo_y - y0 >= mm or win[2] == 0) and (y1 - hi_y >= mm or win[3] == b0["nel"][1]))
            info["pmut_valid"].append(valid)
        keep = np.array(keep, dtype=np.int64)
        npm = dict(pm)
        for key in ("centers", "freq_hz", "delay_s"):
            npm[key] = np.asarray(pm[key])[keep]
        crop["pmut"] = npm if len(keep) else None
        info["pmut_full_index"] = keep
    if rec.get("plane_wave") is not None:
        pw = dict(rec["plane_wave"])
        b = full_boxes[pw["box"]]
        kd = np.asarray(pw["direction"], dtype=np.float64)
        zt = b["origin"][2] + b["extent"][2]
        corners = np.array([[x, y, zt] for x in (b["origin"][0], b["origin"][0] + b["extent"][0])
                            for y in (b["origin"][1], b["origin"][1] + b["extent"][1])])
        pw["x_ref"] = corners[np.argmin(corners @ kd)]
        crop["plane_wave"] = pw
    return crop, info
