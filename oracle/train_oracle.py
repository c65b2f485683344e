"""CPU oracle for the training kernels.

TEST INFRASTRUCTURE ONLY, with the same rules as gridfield_oracle: only
``tests/`` and ``bench.py``'s CPU legs may import it, and only as the checker
or the timed CPU baseline.

A numpy restatement of the reference's training math:
  mlp.py:238-266   forward with the activations backward needs
  mlp.py:269-316   backward (exact parameter gradients)
  batched.py:154-187 grouped_backward (power-of-two segment stacks, as the
                   reference's grouped_forward caches them)
  train.py:130-160 adam_update / regularization_term
  train.py:212-288 photometric_loss_and_grads
It is pinned against fixtures the reference itself wrote
(tests/golden/train.npz; tests/test_train_oracle.py).
"""

from __future__ import annotations

import numpy as np

from .gridfield_oracle import Lattice, _dense, _logistic, _stacks, alpha_of, bin_cells, encode, group

REGULARIZED_LAYERS = ("direction", "color")


def forward_cache(w, b, xe, de, trunk_layers=2):
    """mlp.py:238-266 keeping hs, sigma, feat, g, color."""
    hs = []
    h = np.maximum(_dense(w["trunk0"], b["trunk0"], xe), 0.0)
    hs.append(h)
    for k in range(1, trunk_layers):
        h = np.maximum(_dense(w[f"trunk{k}"], b[f"trunk{k}"], h), 0.0)
        hs.append(h)
    sigma = np.maximum(_dense(w["density"], b["density"], h)[..., 0], 0.0)
    feat = _dense(w["feature"], b["feature"], h)
    g = np.maximum(_dense(w["direction"], b["direction"], np.concatenate([feat, de], axis=-1)), 0.0)
    color = _logistic(_dense(w["color"], b["color"], g))
    return dict(x_enc=xe, d_enc=de, hs=hs, sigma=sigma, feat=feat, g=g, color=color)


def backward(w, c, d_color, d_sigma, width, trunk_layers=2):
    """mlp.py:269-316: gradients of sum(d_color*color + d_sigma*sigma)."""
    gw, gb = {}, {}

    def grad_affine(name, dz, x):
        gw[name] = np.matmul(np.swapaxes(dz, -1, -2), x)
        gb[name] = dz.sum(axis=-2)
        return np.matmul(dz, w[name])

    dz_color = d_color * c["color"] * (1.0 - c["color"])
    dg = grad_affine("color", dz_color, c["g"])
    dz_dir = dg * (c["g"] > 0)
    d_dir_in = grad_affine("direction", dz_dir, np.concatenate([c["feat"], c["d_enc"]], axis=-1))
    dfeat = d_dir_in[..., :width]
    dh = grad_affine("feature", dfeat, c["hs"][-1])
    dz_density = (np.asarray(d_sigma) * (c["sigma"] > 0))[..., None]
    dh = dh + grad_affine("density", dz_density, c["hs"][-1])
    for k in range(trunk_layers - 1, 0, -1):
        dz = dh * (c["hs"][k] > 0)
        dh = grad_affine(f"trunk{k}", dz, c["hs"][k - 1])
    dz = dh * (c["hs"][0] > 0)
    grad_affine("trunk0", dz, c["x_enc"])
    return gw, gb


def grouped_forward_backward(lat: Lattice, positions, directions, d_color, d_sigma):
    """batched.py:120-187 for one batch: group by cell, evaluate each length
    stack with caches, backpropagate upstream gradients given in query order.
    Returns (rgb, sigma) in query order and per-layer gradients stacked over
    all cells (zeros for unqueried cells)."""
    keys = bin_cells(positions, lat.b_min, lat.b_max, lat.res)
    grp = group(keys, lat.n_cells)
    pos_s = np.ascontiguousarray(positions[grp.order])
    dir_s = np.ascontiguousarray(directions[grp.order])
    dc_s, ds_s = d_color[grp.order], d_sigma[grp.order]
    dtype = lat.weights["trunk0"].dtype
    width = lat.weights["trunk0"].shape[-2]
    n = len(grp.order)
    rgb = np.zeros((n, 3), dtype)
    sig = np.zeros(n, dtype)
    gw = {k: np.zeros_like(v) for k, v in lat.weights.items()}
    gb = {k: np.zeros_like(v) for k, v in lat.biases.items()}
    for cells, rows, valid in _stacks(grp.offsets):
        p, d = pos_s[rows].astype(dtype), dir_s[rows].astype(dtype)
        dcol, dsig = dc_s[rows], ds_s[rows]
        if valid is not None:
            p[~valid] = 0.0
            d[~valid] = 0.0
            dcol = dcol.copy()
            dsig = dsig.copy()
            dcol[~valid] = 0.0
            dsig[~valid] = 0.0
        w = {k: v[cells] for k, v in lat.weights.items()}
        b = {k: v[cells] for k, v in lat.biases.items()}
        c = forward_cache(w, b, encode(p, lat.pos_freqs, lat.include_raw), encode(d, lat.dir_freqs, lat.include_raw),
                          lat.trunk_layers)
        if valid is None:
            rgb[rows.ravel()] = c["color"].reshape(-1, 3)
            sig[rows.ravel()] = c["sigma"].reshape(-1)
        else:
            rgb[rows[valid]] = c["color"][valid]
            sig[rows[valid]] = c["sigma"][valid]
        bw, bb = backward(w, c, dcol, dsig, width, lat.trunk_layers)
        for k in gw:
            gw[k][cells] = bw[k]
            gb[k][cells] = bb[k]
    return rgb[grp.inverse], sig[grp.inverse], gw, gb


def photometric_loss_and_grads(lat: Lattice, pos, dirs, ray_index, slot, deltas, n_rays, k, gt, background,
                               reg_weight=0.0, sigma_noise=None):
    """train.py:212-288 (two passes: forward for colours, then backward with
    the compositing gradients; the network math is identical both times)."""
    dtype = lat.weights["trunk0"].dtype
    q = len(pos)
    colors, sigmas, _, _ = grouped_forward_backward(lat, pos, dirs, np.zeros((q, 3), dtype), np.zeros(q, dtype))
    noise_mask = None
    if sigma_noise is not None:
        shifted = sigmas + sigma_noise.astype(dtype)
        noise_mask = shifted > 0
        sigmas = np.maximum(shifted, 0.0)
    deltas = deltas.astype(dtype)
    alpha = np.zeros((n_rays, k), dtype)
    color = np.zeros((n_rays, k, 3), dtype)
    alpha[ray_index, slot] = alpha_of(sigmas, deltas[ray_index])
    color[ray_index, slot] = colors
    trans = np.cumprod(1.0 - alpha, axis=1)
    t_before = np.concatenate([np.ones_like(trans[:, :1]), trans[:, :-1]], axis=1)
    weights = t_before * alpha
    bg = np.asarray(background, dtype=dtype)
    pred = (weights[..., None] * color).sum(axis=1) + trans[:, -1:] * bg[None, :]
    resid = pred - gt.astype(dtype)
    loss = float((resid.astype(np.float64) ** 2).sum(axis=-1).mean())
    reg = None
    if reg_weight > 0.0:
        value, reg = regularization_term(lat, reg_weight)
        loss += value
    dpred = (2.0 / n_rays) * resid
    rest = np.empty_like(color)
    rest[:, -1] = bg
    for i in range(k - 2, -1, -1):
        a = alpha[:, i + 1 : i + 2]
        rest[:, i] = a * color[:, i + 1] + (1.0 - a) * rest[:, i + 1]
    d_alpha = (dpred[:, None, :] * t_before[..., None] * (color - rest)).sum(axis=-1)
    d_color_q = (weights[..., None] * dpred[:, None, :])[ray_index, slot]
    d_sigma_q = (d_alpha * deltas[:, None] * (1.0 - alpha))[ray_index, slot]
    if noise_mask is not None:
        d_sigma_q = d_sigma_q * noise_mask
    _, _, gw, gb = grouped_forward_backward(lat, pos, dirs, d_color_q, d_sigma_q)
    if reg is not None:
        for name in REGULARIZED_LAYERS:
            gw[name] = gw[name] + reg[0][name]
            gb[name] = gb[name] + reg[1][name]
    return loss, gw, gb


def regularization_term(lat: Lattice, weight: float):
    """train.py:146-160."""
    value = 0.0
    gw, gb = {}, {}
    for name in REGULARIZED_LAYERS:
        w, b = lat.weights[name], lat.biases[name]
        value += float((w.astype(np.float64) ** 2).sum() + (b.astype(np.float64) ** 2).sum())
        gw[name] = 2.0 * weight * w
        gb[name] = 2.0 * weight * b
    return weight * value, (gw, gb)


def adam_update(arrays, grads, m, v, step, lr, b1=0.9, b2=0.999, eps=1e-8):
    """train.py:130-143 over matching lists of arrays, in place; returns the
    new step count."""
    step += 1
    bc1 = 1.0 - b1**step
    bc2 = 1.0 - b2**step
    for p, g, mm, vv in zip(arrays, grads, m, v):
        mm *= b1
        mm += (1.0 - b1) * g
        vv *= b2
        vv += (1.0 - b2) * g * g
        p -= lr * (mm / bc1) / (np.sqrt(vv / bc2) + eps)
    return step
