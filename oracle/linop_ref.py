"""numpy restatement of the reference operator algebra (TEST ORACLE ONLY).

Restates /root/reference/pkg/src/conegraph/linop.py:
  conv_full        linop.py:41-50   (direct below FFT_CROSSOVER=512, FFT above)
  corr_valid       linop.py:53-64
  _forward         linop.py:210-231
  _adjoint         linop.py:234-260
  materialize      linop.py:368-384
Extensions required by the north star (no reference counterpart): Conv2D
(full 2-D convolution, adjoint = valid 2-D correlation) and Kron
(np.kron convention).  Dispatch is by class name so the oracle walks the
product package's expression trees without importing the product.
"""

from __future__ import annotations

import numpy as np
import scipy.fft
import scipy.signal

FFT_CROSSOVER = 512  # linop.py:36


def conv_full(kernel: np.ndarray, x: np.ndarray, method: str = "auto") -> np.ndarray:
    """linop.py:41-50 -- full 1-d convolution, length k+n-1."""
    if method == "auto":
        method = "fft" if max(len(kernel), len(x)) > FFT_CROSSOVER else "direct"
    if method == "direct":
        return np.convolve(kernel, x)
    out_len = len(kernel) + len(x) - 1
    nfft = scipy.fft.next_fast_len(out_len)
    spec = np.fft.rfft(kernel, nfft) * np.fft.rfft(x, nfft)
    return np.fft.irfft(spec, nfft)[:out_len]


def corr_valid(kernel: np.ndarray, y: np.ndarray, method: str = "auto") -> np.ndarray:
    """linop.py:53-64 -- valid correlation out[j] = sum_i kernel[i] y[j+i]."""
    if method == "auto":
        method = "fft" if max(len(kernel), len(y)) > FFT_CROSSOVER else "direct"
    if method == "direct":
        return np.correlate(y, kernel, mode="valid")
    k = len(kernel)
    full = conv_full(kernel[::-1], y, method="fft")
    return full[k - 1:len(y)]


def conv2d_full(kernel: np.ndarray, x: np.ndarray) -> np.ndarray:
    """Full 2-d convolution (north-star Conv2D leaf); x, kernel 2-d."""
    return scipy.signal.convolve(x, kernel, mode="full", method="auto")


def corr2d_valid(kernel: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Adjoint of conv2d_full: valid 2-d correlation."""
    return scipy.signal.correlate(y, kernel, mode="valid", method="auto")


def _name(e) -> str:
    return type(e).__name__


def forward(e, x: np.ndarray) -> np.ndarray:
    """linop.py:210-231 (_forward) plus Conv2D/Kron extensions."""
    x = np.asarray(x, dtype=np.float64)
    k = _name(e)
    if k == "DenseMatrix":
        return e.values @ x
    if k == "Conv1D":
        return conv_full(e.kernel, x)
    if k == "Conv2D":
        h, w = e.image_shape
        return conv2d_full(e.kernel, x.reshape(h, w)).ravel()
    if k == "Identity":
        return x
    if k == "Scale":
        return e.alpha * forward(e.child, x)
    if k == "Sum":
        return forward(e.left, x) + forward(e.right, x)
    if k == "Compose":
        return forward(e.left, forward(e.right, x))
    if k == "VStack":
        return np.concatenate([forward(c, x) for c in e.children])
    if k == "AdjointOf":
        return adjoint(e.child, x)
    if k == "SparseMatrix":
        return e.matrix @ x
    if k == "ZeroOp":
        return np.zeros(e.rows)
    if k == "Kron":
        return _kron_apply(e.left, e.right, x, forward)
    raise TypeError(f"oracle: unknown expression {k}")


def adjoint(e, y: np.ndarray) -> np.ndarray:
    """linop.py:234-260 (_adjoint) plus Conv2D/Kron extensions."""
    y = np.asarray(y, dtype=np.float64)
    k = _name(e)
    if k == "DenseMatrix":
        return e.values.T @ y
    if k == "Conv1D":
        return corr_valid(e.kernel, y)
    if k == "Conv2D":
        h, w = e.image_shape
        kh, kw = e.kernel.shape
        return corr2d_valid(e.kernel, y.reshape(h + kh - 1, w + kw - 1)).ravel()
    if k == "Identity":
        return y
    if k == "Scale":
        return e.alpha * adjoint(e.child, y)
    if k == "Sum":
        return adjoint(e.left, y) + adjoint(e.right, y)
    if k == "Compose":
        return adjoint(e.right, adjoint(e.left, y))
    if k == "VStack":
        out = np.zeros(e.cols)
        off = 0
        for c in e.children:
            out += adjoint(c, y[off:off + c.rows])
            off += c.rows
        return out
    if k == "AdjointOf":
        return forward(e.child, y)
    if k == "SparseMatrix":
        return e.matrix.T @ y
    if k == "ZeroOp":
        return np.zeros(e.cols)
    if k == "Kron":
        return _kron_apply(e.left, e.right, y, adjoint)
    raise TypeError(f"oracle: unknown expression {k}")


def _kron_apply(L, R, x, app):
    """(L (x) R) x with np.kron index convention; app = forward or adjoint."""
    if app is forward:
        p, q = L.rows, L.cols
        r, s = R.rows, R.cols
    else:
        p, q = L.cols, L.rows
        r, s = R.cols, R.rows
    X = x.reshape(q, s)
    Z = np.stack([app(R, X[j]) for j in range(q)]) if q else np.zeros((0, r))
    out = np.stack([app(L, Z[:, kk]) for kk in range(r)], axis=1) if r else np.zeros((p, 0))
    return out.reshape(p * r)


def materialize(e) -> np.ndarray:
    """linop.py:368-384 -- column j is forward(e_j) (small operators only)."""
    m, n = e.rows, e.cols
    out = np.zeros((m, n))
    unit = np.zeros(n)
    for j in range(n):
        unit[j] = 1.0
        out[:, j] = forward(e, unit)
        unit[j] = 0.0
    return out
