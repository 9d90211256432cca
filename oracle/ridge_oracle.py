"""CPU restatement of the reference ridge head — TEST INFRASTRUCTURE / CPU
BASELINE ONLY (bench.py's config-1 CPU leg and tests; never the product).

Follows /root/reference/pkg/src/gridrocket/ridge.py:100-157 with numpy and
scipy's LAPACK Cholesky: population-statistics standardisation (zero scales
become 1, :125-129), the primal system (X'X + alpha I) W = X'Y when
n_features <= n_instances else the dual (XX' + alpha I) A = Y, W = X'A
(:100-122), one-vs-rest +1/-1 targets centred by their column means
(:132-157), argmax prediction with ties to the lowest class (:191-197).
Pinned against the reference's own fits in tests/golden/ridge.npz."""

import numpy as np
from scipy.linalg import cho_factor, cho_solve


def solve_penalized(X, Y, alpha):
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    single = Y.ndim == 1
    if single:
        Y = Y[:, None]
    n, f = X.shape
    if f <= n:
        gram = X.T @ X
        gram[np.diag_indices_from(gram)] += alpha
        W = cho_solve(cho_factor(gram), X.T @ Y)
    else:
        outer = X @ X.T
        outer[np.diag_indices_from(outer)] += alpha
        W = X.T @ cho_solve(cho_factor(outer), Y)
    return W[:, 0] if single else W


def fit(features, labels, alpha=1.0):
    """(weights, intercepts, means, scales, class_names) of the reference's
    ridge.fit."""
    X = np.asarray(features, dtype=np.float64)
    labels = [str(v) for v in labels]
    names = sorted(set(labels))
    means = X.mean(axis=0)
    scales = X.std(axis=0)
    scales[~(scales > 0.0)] = 1.0
    Xs = (X - means) / scales
    index = {c: i for i, c in enumerate(names)}
    Y = np.full((X.shape[0], len(names)), -1.0)
    for row, lab in enumerate(labels):
        Y[row, index[lab]] = 1.0
    intercepts = Y.mean(axis=0)
    W = solve_penalized(Xs, Y - intercepts, alpha)
    return W, intercepts, means, scales, names


def predict(model, features):
    W, intercepts, means, scales, names = model
    X = np.asarray(features, dtype=np.float64)
    scores = ((X - means) / scales) @ W + intercepts
    return np.asarray([names[i] for i in np.argmax(scores, axis=1)])
