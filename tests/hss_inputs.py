"""Inputs of /root/reference/proj/tests/test_hss.cpp:13-31 and the testgen
kernels it uses (testgen.cpp:132-148, 216-253), built with numpy from a
library's own Rng (oracle or product: same mt19937_64 stream)."""
import numpy as np


def block_diagonal(rng, blocks, b):  # test_hss.cpp:13-18
    M = np.zeros((blocks * b, blocks * b))
    for t in range(blocks):
        M[t * b:(t + 1) * b, t * b:(t + 1) * b] = rng.gaussian_matrix(b, b)
    return M


def tridiagonal(n, rng):  # test_hss.cpp:20-30 (draw order: diag, upper, lower)
    M = np.zeros((n, n))
    for i in range(n):
        M[i, i] = 2 + rng.uniform()
        if i + 1 < n:
            M[i, i + 1] = -1 + 0.1 * rng.uniform()
            M[i + 1, i] = -1 + 0.1 * rng.uniform()
    return M


def cauchy_kernel(n):  # testgen.cpp:247-253
    i = np.arange(n, dtype=np.float64)
    return 1.0 / (i[:, None] + 0.5 - i[None, :])


def gravity_kernel(m, n):  # testgen.cpp:216-230, 243
    x = (np.arange(m) + 0.5) / m
    y = (np.arange(n) + 0.5) / n
    d = x[:, None] - y[None, :]
    return np.power(1.0 + d * d, -1.5)


def gen_fd_inverse(m, n):  # testgen.cpp:132-148
    g = 2
    while g * g < m + n:
        g += 1
    N = g * g
    A = np.zeros((N, N))
    for x in range(g):
        for y in range(g):
            p = x * g + y
            A[p, p] = 4.0
            if x > 0:
                A[p, p - g] = -1.0
            if x + 1 < g:
                A[p, p + g] = -1.0
            if y > 0:
                A[p, p - 1] = -1.0
            if y + 1 < g:
                A[p, p + 1] = -1.0
    return np.linalg.inv(A)[:m, N - n:]
