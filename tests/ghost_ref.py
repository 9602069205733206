"""Dense numpy restatement of tt_ghosted (cases.cpp:298-344) for the ghost-cell tests:
the pad matrices of reconstruction.hpp:473-485 and the rank-additive Dirichlet strips."""
import numpy as np

G = 3


def pad_matrix(n, dirichlet):
    p = np.zeros((n + 2 * G, n))
    for i in range(n + 2 * G):
        if dirichlet:
            if G <= i < n + G:
                p[i, i - G] = 1.0
        else:
            p[i, (i - G) % n] = 1.0
    return p


def dense_ghosted(a, dir_x, dir_y, strip_x, strip_y):
    nx, ny = a.shape
    out = pad_matrix(nx, dir_x) @ a @ pad_matrix(ny, dir_y).T
    if dir_x:
        rows = list(range(G)) + list(range(nx + G, nx + 2 * G))
        out[rows, :] += strip_x
    if dir_y:
        cols = list(range(G)) + list(range(ny + G, ny + 2 * G))
        s = np.array(strip_y, dtype=float)
        if dir_x:
            s[:G, :] = 0.0
            s[nx + G:, :] = 0.0
        out[:, cols] += s
    return out


def case(rng, nx, ny, r):
    cx = rng.standard_normal((nx, r))
    cy = rng.standard_normal((r, ny))
    sx = rng.standard_normal((2 * G, ny + 2 * G))
    sy = rng.standard_normal((nx + 2 * G, 2 * G))
    return cx, cy, sx, sy
