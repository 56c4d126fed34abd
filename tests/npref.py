"""Independent numpy restatement used to pin the C++ oracle (test-only).

Written from the reference's documented maths, not from
the oracle's code: direct sums instead of FFTs wherever sizes allow.
"""
import numpy as np


def support(shape, tau, nd):
    pts = np.stack(np.meshgrid(*[np.arange(-tau, tau + 1)] * nd, indexing="ij"), -1).reshape(-1, nd)
    if shape == 1:
        pts = pts[(pts ** 2).sum(1) <= tau * tau]
    return pts


def calib_full_matrix(calib, offs):
    """C_full: rows = all shifts y with any sample (E+2tau per axis), cols (q, s): x_q[y - n_s]."""
    q = calib.shape[0]
    dims = calib.shape[1:]
    tau = int(np.abs(offs).max()) if offs.size else 0
    nd = len(dims)
    ys = np.stack(np.meshgrid(*[np.arange(-tau, e + tau) for e in dims], indexing="ij"), -1).reshape(-1, nd)
    rows = []
    lam = offs.shape[0]
    C = np.zeros((ys.shape[0], q * lam), dtype=np.complex128)
    for s in range(lam):
        src = ys - offs[s]
        ok = np.all((src >= 0) & (src < np.array(dims)), axis=1)
        idx = tuple(src[ok].T)
        for c in range(q):
            C[ok, c * lam + s] = calib[c][idx]
    del rows
    return C


def field_direct(W, offs, q, dims):
    """G_pq(x) = sum_{s,t} W[(q,s),(p,t)] exp(-i 2 pi (m_t - n_s) x), returned [j,p,q]."""
    lam = offs.shape[0]
    nd = len(dims)
    xs = np.stack(np.meshgrid(*[(np.arange(n) - n // 2) / n for n in dims], indexing="ij"), -1).reshape(-1, nd)
    E = np.exp(2j * np.pi * xs @ offs.T)          # N x lam : e^{+i 2 pi n_s x}
    G = np.zeros((xs.shape[0], q, q), dtype=np.complex128)
    for p in range(q):
        for qq in range(q):
            blk = W[qq * lam:(qq + 1) * lam, p * lam:(p + 1) * lam]   # [s, t]
            G[:, p, qq] = np.einsum("js,st,jt->j", E, blk, E.conj())
    return G


def power(B, iters):
    n, q, _ = B.shape
    v = np.full((n, q), 1 / np.sqrt(q), dtype=np.complex128)
    for _ in range(iters):
        w = np.einsum("jpq,jq->jp", B, v)
        v = w / np.linalg.norm(w, axis=1, keepdims=True)
    val = np.real(np.einsum("jp,jpq,jq->j", v.conj(), B, v))
    return v, val


def centered_dft_matrix(n_out, n_in, c_out, c_in, sign, scale=1.0):
    j = np.arange(n_out)[:, None] - c_out
    a = np.arange(n_in)[None, :] - c_in
    return scale * np.exp(sign * 2j * np.pi * j * a / n_out)
