"""Seeded synthetic input generator shared by the oracle tests and the CUDA path.

It holds none of the method's arithmetic: it only draws and splats shapes.  Recipe
(after SURVEY §8d): the paper's workload is natural grayscale images of 240x400 to
1920x1200 with ~2200 keypoints at 480x640; the generator imitates that
density with, per 640x480 of area, 200 additive shapes (half axis-aligned rectangles with sides
U(6, 60), half disks with radius U(3, 30), amplitude U(-0.25, 0.25)) and 4000 Gaussian blobs
(std log-uniform in [1.2, 10] px, amplitude U(-0.35, 0.35)) on a 0.5 background, plus N(0, 0.01)
noise, clipped to [0, 1] and stored as float32 (values in [0, 1] as SPEC S:L455 scales images).
Seed of image i is 1234 + i (numpy default_rng).
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 1234


def synth_image(width: int, height: int, seed: int = BASE_SEED, complexity: float = 1.0) -> np.ndarray:
    """One synthetic image as float32 (height, width) in [0, 1].

    ``complexity`` scales the number of shapes and blobs per area (1.0 = the recipe above); the stage-timing
    sweep uses several values per size, like the paper's "6 images of varying complexity in each
    dimension"."""
    W, H = int(width), int(height)
    rng = np.random.default_rng(seed)
    scale = (W * H) / (640.0 * 480.0) * float(complexity)
    n_shapes = max(1, int(round(200 * scale)))
    n_blobs = max(1, int(round(4000 * scale)))
    img = np.full((H, W), 0.5, dtype=np.float64)

    # --- shapes (parameters drawn in one fixed order) ---
    kind = rng.integers(0, 2, n_shapes)               # 0 rectangle, 1 disk
    cx = rng.uniform(0, W, n_shapes)
    cy = rng.uniform(0, H, n_shapes)
    sw = rng.uniform(6, 60, n_shapes)
    sh = rng.uniform(6, 60, n_shapes)
    rad = rng.uniform(3, 30, n_shapes)
    amp = rng.uniform(-0.25, 0.25, n_shapes)
    for i in range(n_shapes):
        if kind[i] == 0:
            x0 = int(np.clip(np.floor(cx[i] - sw[i] / 2), 0, W)); x1 = int(np.clip(np.ceil(cx[i] + sw[i] / 2), 0, W))
            y0 = int(np.clip(np.floor(cy[i] - sh[i] / 2), 0, H)); y1 = int(np.clip(np.ceil(cy[i] + sh[i] / 2), 0, H))
            img[y0:y1, x0:x1] += amp[i]
        else:
            r = rad[i]
            x0 = int(max(0, np.floor(cx[i] - r))); x1 = int(min(W, np.ceil(cx[i] + r) + 1))
            y0 = int(max(0, np.floor(cy[i] - r))); y1 = int(min(H, np.ceil(cy[i] + r) + 1))
            if x1 <= x0 or y1 <= y0:
                continue
            yy, xx = np.mgrid[y0:y1, x0:x1]
            m = (xx - cx[i]) ** 2 + (yy - cy[i]) ** 2 <= r * r
            img[y0:y1, x0:x1] += amp[i] * m

    # --- Gaussian blobs ---
    bx = rng.uniform(0, W, n_blobs)
    by = rng.uniform(0, H, n_blobs)
    bs = np.exp(rng.uniform(np.log(1.2), np.log(10.0), n_blobs))
    ba = rng.uniform(-0.35, 0.35, n_blobs)
    for i in range(n_blobs):
        r = int(np.ceil(3 * bs[i]))
        xc, yc = int(np.floor(bx[i])), int(np.floor(by[i]))
        x0, x1 = max(0, xc - r), min(W, xc + r + 1)
        y0, y1 = max(0, yc - r), min(H, yc + r + 1)
        if x1 <= x0 or y1 <= y0:
            continue
        gx = np.exp(-((np.arange(x0, x1) - bx[i]) ** 2) / (2 * bs[i] ** 2))
        gy = np.exp(-((np.arange(y0, y1) - by[i]) ** 2) / (2 * bs[i] ** 2))
        img[y0:y1, x0:x1] += ba[i] * np.outer(gy, gx)

    img += rng.normal(0.0, 0.01, (H, W))
    np.clip(img, 0.0, 1.0, out=img)
    return img.astype(np.float32)


def synth_batch(n: int, width: int, height: int, first: int = 0, distinct: int | None = None) -> np.ndarray:
    """n images (n, H, W) float32.  Image i uses seed 1234 + (first + i).

    With ``distinct`` = d < n, only d images are generated and image i is derived from image
    i mod d by an integer translation (np.roll) and flips determined by i // d — keeping the
    statistics while bounding generation time for large batches."""
    if distinct is None or distinct >= n:
        return np.stack([synth_image(width, height, BASE_SEED + first + i) for i in range(n)])
    base = [synth_image(width, height, BASE_SEED + first + i) for i in range(distinct)]
    out = np.empty((n, height, width), np.float32)
    for i in range(n):
        j, v = i % distinct, i // distinct
        im = base[j]
        if v:
            im = np.roll(im, (37 * v) % height, axis=0)
            im = np.roll(im, (101 * v) % width, axis=1)
            if v & 1:
                im = im[:, ::-1]
            if v & 2:
                im = im[::-1, :]
        out[i] = im
    return out
