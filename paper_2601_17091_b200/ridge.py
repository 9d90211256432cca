"""Ridge head on the GPU: the reference's closed-form ridge
(/root/reference/pkg/src/gridrocket/ridge.py:100-242) in float64 torch, so
the features the transform leaves in HBM never travel to the host.

Same API and arithmetic as the reference: features are standardised with
population statistics (zero scales become 1, ridge.py:125-129); the normal
equations (X'X + alpha I) W = X'Y are solved through a Cholesky
factorisation in the primal when n_features <= n_instances and in the dual
(XX' + alpha I) A = Y, W = X'A otherwise (ridge.py:100-122); one-vs-rest
targets are +1/-1 with the column means as intercepts (ridge.py:132-157);
ties in predict resolve to the lowest class index (ridge.py:193-199).
Results match the reference's scipy (LAPACK) solve to float64 rounding, not
bit for bit.

For series-sharded features (one process per GPU, paper_2601_17091_b200.
distributed) fit_sharded all-reduces the column sums and the primal Gram
partials X_r'X_r (NCCL over NVLink on GPUs), or all-gathers the rows for the
dual — the only collective of the pipeline.
"""

from dataclasses import dataclass

import numpy as np
import torch

from .binio import read_array, read_header, read_str, read_values, write_array, write_header, write_str, write_values

MODEL_MAGIC = b"RKRM"
MODEL_VERSION = 1


@dataclass
class RidgeModel:
    """Linear model with the standardisation statistics baked in
    (ridge.py:30-47); arrays are float64 numpy."""

    weights: np.ndarray
    intercepts: np.ndarray
    feature_means: np.ndarray
    feature_scales: np.ndarray
    alpha: float
    class_names: list | None = None

    @property
    def n_features(self) -> int:
        return self.weights.shape[0]

    def save(self, path) -> None:
        """RKRM v1, the reference's model file (ridge.py:49-67): header,
        QQdB (n_features, n_outputs, alpha, has_classes), float64 weights,
        intercepts, means, scales, then the class names."""
        weights = np.asarray(self.weights, dtype=np.float64)
        n_features, n_outputs = weights.shape
        with open(path, "wb") as f:
            write_header(f, MODEL_MAGIC, MODEL_VERSION)
            write_values(f, "QQdB", n_features, n_outputs, float(self.alpha), 1 if self.class_names is not None else 0)
            for arr in (weights, self.intercepts, self.feature_means, self.feature_scales):
                write_array(f, np.asarray(arr, dtype=np.float64))
            for name in self.class_names or ():
                write_str(f, name)

    @classmethod
    def load(cls, path) -> "RidgeModel":
        """Read an RKRM v1 file (ridge.py:69-88); FormatError on a bad file."""
        with open(path, "rb") as f:
            read_header(f, MODEL_MAGIC, MODEL_VERSION)
            n_features, n_outputs, alpha, has_classes = read_values(f, "QQdB")
            nf, no = int(n_features), int(n_outputs)
            weights = read_array(f, np.float64, nf * no).reshape(nf, no)
            intercepts = read_array(f, np.float64, no)
            means = read_array(f, np.float64, nf)
            scales = read_array(f, np.float64, nf)
            names = [read_str(f) for _ in range(no)] if has_classes else None
        return cls(weights=weights, intercepts=intercepts, feature_means=means, feature_scales=scales,
                   alpha=float(alpha), class_names=names)


def _device_of(features, device):
    if device is not None:
        return torch.device(device)
    if isinstance(features, torch.Tensor):
        return features.device
    return torch.device("cuda" if torch.cuda.is_available() else "cpu")


def _as_matrix(features, device=None) -> torch.Tensor:
    """float64 (n, F) tensor on the working device (ridge.py:91-97)."""
    dev = _device_of(features, device)
    values = features
    if not isinstance(features, (torch.Tensor, np.ndarray)) and hasattr(features, "values"):
        values = features.values  # FeatureMatrix
    if isinstance(values, torch.Tensor):
        X = values.to(device=dev, dtype=torch.float64)
    else:
        X = torch.as_tensor(np.asarray(values, dtype=np.float64), device=dev)
    if X.ndim != 2:
        raise ValueError("features must be a 2-D matrix")
    if not bool(torch.isfinite(X).all()):
        raise ValueError("features contain non-finite values")
    return X


def _chol_solve(A: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
    L, info = torch.linalg.cholesky_ex(A)
    if int(info) != 0:
        raise np.linalg.LinAlgError("penalised system is not positive definite")
    return torch.cholesky_solve(B, L)


def _gram_rows(X: torch.Tensor, blocks: int = 4) -> torch.Tensor:
    """X X^T using its symmetry: the upper block triangle of a `blocks` x
    `blocks` split (10 of 16 GEMM blocks for 4), mirrored.  The n x n Gram of
    the dual solve is the FP64-GEMM-bound step of a ridge fit."""
    n = X.shape[0]
    if n < 512 or X.device.type != "cuda":
        return X @ X.T
    edges = [n * i // blocks for i in range(blocks + 1)]
    G = torch.empty((n, n), dtype=X.dtype, device=X.device)
    for i in range(blocks):
        a0, a1 = edges[i], edges[i + 1]
        Xa = X[a0:a1]
        for j in range(i, blocks):
            b0, b1 = edges[j], edges[j + 1]
            blk = Xa @ X[b0:b1].T
            G[a0:a1, b0:b1] = blk
            if j != i:
                G[b0:b1, a0:a1] = blk.T
    return G


def solve_penalized(X, Y, alpha: float):
    """Solve (X'X + alpha I) W = X'Y in float64 (ridge.py:100-122)."""
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    X = torch.as_tensor(X, dtype=torch.float64)
    Y = torch.as_tensor(Y, dtype=torch.float64, device=X.device)
    single = Y.ndim == 1
    if single:
        Y = Y[:, None]
    n, f = X.shape
    if f <= n:
        gram = _gram_rows(X.T)
        gram.diagonal().add_(alpha)
        W = _chol_solve(gram, X.T @ Y)
    else:
        outer = _gram_rows(X)
        outer.diagonal().add_(alpha)
        W = X.T @ _chol_solve(outer, Y)
    return W[:, 0] if single else W


def _standardize(X: torch.Tensor):
    """Population mean / std per column; non-positive scales become 1
    (ridge.py:125-129)."""
    means = X.mean(dim=0)
    scales = X.std(dim=0, correction=0)
    scales = torch.where(scales > 0.0, scales, torch.ones_like(scales))
    return (X - means) / scales, means, scales


def _targets(labels, n):
    labels = [str(lab) for lab in labels]
    if len(labels) != n:
        raise ValueError("one label per instance is required")
    class_names = sorted(set(labels))
    if len(class_names) < 2:
        raise ValueError("classification needs at least two classes")
    index = {name: i for i, name in enumerate(class_names)}
    Y = np.full((n, len(class_names)), -1.0)
    for row, lab in enumerate(labels):
        Y[row, index[lab]] = 1.0
    return Y, class_names


def _model(W, intercepts, means, scales, alpha, class_names):
    return RidgeModel(
        weights=W.detach().cpu().numpy(),
        intercepts=np.asarray(intercepts, dtype=np.float64),
        feature_means=means.detach().cpu().numpy(),
        feature_scales=scales.detach().cpu().numpy(),
        alpha=float(alpha),
        class_names=class_names,
    )


def fit(features, labels, alpha: float = 1.0, device=None) -> RidgeModel:
    """One-vs-rest ridge classifier on standardised features
    (ridge.py:132-157)."""
    X = _as_matrix(features, device)
    if X.shape[0] < 2:
        raise ValueError("at least two instances are required")
    Y, class_names = _targets(labels, X.shape[0])
    Xs, means, scales = _standardize(X)
    intercepts = Y.mean(axis=0)
    Yt = torch.as_tensor(Y - intercepts, device=X.device)
    W = solve_penalized(Xs, Yt, alpha)
    return _model(W, intercepts, means, scales, alpha, class_names)


def fit_regression(features, targets, alpha: float = 1.0, device=None) -> RidgeModel:
    """Ridge regressor on standardised features (ridge.py:160-178)."""
    X = _as_matrix(features, device)
    if X.shape[0] < 2:
        raise ValueError("at least two instances are required")
    y = np.asarray(targets, dtype=np.float64)
    if y.shape != (X.shape[0],):
        raise ValueError("one target per instance is required")
    Xs, means, scales = _standardize(X)
    intercept = y.mean()
    w = solve_penalized(Xs, torch.as_tensor(y - intercept, device=X.device), alpha)
    return _model(w[:, None], np.array([intercept]), means, scales, alpha, None)


def predict_scores(model: RidgeModel, features, device=None) -> np.ndarray:
    """Standardised features times weights plus intercepts (ridge.py:181-188)."""
    X = _as_matrix(features, device)
    if X.shape[1] != model.n_features:
        raise ValueError(f"model expects {model.n_features} features, got {X.shape[1]}")
    dev = X.device
    Xs = (X - torch.as_tensor(model.feature_means, device=dev)) / torch.as_tensor(model.feature_scales, device=dev)
    scores = Xs @ torch.as_tensor(model.weights, device=dev) + torch.as_tensor(model.intercepts, device=dev)
    return scores.cpu().numpy()


def predict(model: RidgeModel, features, device=None) -> np.ndarray:
    """Class labels; score ties resolve to the lowest class index
    (ridge.py:191-198)."""
    if model.class_names is None:
        raise ValueError("model was fit for regression; use predict_values")
    picks = np.argmax(predict_scores(model, features, device), axis=1)
    return np.asarray([model.class_names[i] for i in picks])


def predict_values(model: RidgeModel, features, device=None) -> np.ndarray:
    """Regression predictions (ridge.py:201-203)."""
    return predict_scores(model, features, device)[:, 0]


def accuracy(predicted, truth) -> float:
    """Fraction of matching labels (ridge.py:206-214)."""
    predicted = [str(p) for p in predicted]
    truth = [str(t) for t in truth]
    if len(predicted) != len(truth):
        raise ValueError("prediction and truth lengths differ")
    if not truth:
        raise ValueError("cannot score an empty label set")
    return sum(1 for p, t in zip(predicted, truth) if p == t) / len(truth)


def select_alpha(features, labels, alphas, val_fraction: float = 0.25, seed: int = 0, device=None):
    """Pick alpha on a seeded validation split (ridge.py:216-242): the same
    Philox permutation, so the same split as the reference."""
    X = _as_matrix(features, device)
    labels = [str(lab) for lab in labels]
    if not 0.0 < val_fraction < 1.0:
        raise ValueError("val_fraction must be in (0, 1)")
    rng = np.random.Generator(np.random.Philox(key=np.uint64(seed)))
    order = rng.permutation(X.shape[0])
    n_val = max(1, int(round(val_fraction * X.shape[0])))
    val_idx, train_idx = order[:n_val], order[n_val:]
    if train_idx.size < 2:
        raise ValueError("not enough instances left for training")
    tr = torch.as_tensor(train_idx, device=X.device)
    va = torch.as_tensor(val_idx, device=X.device)
    train_labels = [labels[i] for i in train_idx]
    val_labels = [labels[i] for i in val_idx]
    scores, best = {}, None
    for alpha in alphas:
        model = fit(X[tr], train_labels, alpha=alpha)
        acc = accuracy(predict(model, X[va]), val_labels)
        scores[alpha] = acc
        if best is None or acc > scores[best]:
            best = alpha
    return best, scores


def fit_sharded(local_features, local_labels, alpha: float = 1.0, group=None, device=None) -> RidgeModel:
    """fit() over row shards held by the ranks of a torch.distributed group.

    Column sums and sums of squares are all-reduced for the standardisation;
    the primal Gram X'X + alpha I and X'Y are all-reduced from per-rank
    partials (F x F, independent of the row count), or — when the features
    outnumber the rows — the standardised rows are all-gathered for the dual
    system.  Every rank returns the same model, equal to fit() on the
    concatenated rows up to float64 rounding.
    """
    import torch.distributed as dist

    X = _as_matrix(local_features, device)
    labels = [str(lab) for lab in local_labels]
    world = dist.get_world_size(group)
    counts = [None] * world
    dist.all_gather_object(counts, (X.shape[0], labels), group=group)
    n = sum(c for c, _ in counts)
    all_labels = [lab for _, labs in counts for lab in labs]
    if n < 2:
        raise ValueError("at least two instances are required")
    Yall, class_names = _targets(all_labels, n)
    intercepts = Yall.mean(axis=0)
    start = sum(c for c, _ in counts[: dist.get_rank(group)])
    Y = torch.as_tensor(Yall[start : start + X.shape[0]] - intercepts, device=X.device)
    # population mean / std from all-reduced moments (two-pass: mean first)
    s1 = X.sum(dim=0)
    dist.all_reduce(s1, group=group)
    means = s1 / n
    s2 = ((X - means) ** 2).sum(dim=0)
    dist.all_reduce(s2, group=group)
    scales = torch.sqrt(s2 / n)
    scales = torch.where(scales > 0.0, scales, torch.ones_like(scales))
    Xs = (X - means) / scales
    f = X.shape[1]
    if f <= n:
        gram = _gram_rows(Xs.T)
        rhs = Xs.T @ Y
        dist.all_reduce(gram, group=group)
        dist.all_reduce(rhs, group=group)
        gram.diagonal().add_(alpha)
        W = _chol_solve(gram, rhs)
    else:
        rows = [torch.empty((c, f), dtype=torch.float64, device=X.device) for c, _ in counts]
        dist.all_gather(rows, Xs.contiguous(), group=group)
        Xall = torch.cat(rows, dim=0)
        Yfull = torch.as_tensor(Yall - intercepts, device=X.device)
        W = solve_penalized(Xall, Yfull, alpha)
    return _model(W, intercepts, means, scales, alpha, class_names)
