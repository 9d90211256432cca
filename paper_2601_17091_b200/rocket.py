"""sklearn-style ROCKET front end: ``Rocket(num_kernels, seed).fit(X).transform(X)``.

``fit`` draws the bank on the host with the reference's generator
(kernels.generate_bank, reference kernels.py:243-308) from the training
data's shape; ``transform`` runs the B200 kernels (engine.transform).
"""

import numpy as np

from .engine import GridLimits, device_bank, transform
from .kernels import GenOptions, generate_bank


class Rocket:
    def __init__(self, num_kernels=10_000, seed=0, center_weights=True, mode="exact", device=0,
                 limits: GridLimits | None = None):
        self.num_kernels = int(num_kernels)
        self.seed = int(seed)
        self.center_weights = bool(center_weights)
        self.mode = mode
        self.device = int(device)
        self.limits = limits
        self.bank_ = None

    def fit(self, X, y=None):
        values = np.asarray(getattr(X, "values", X))
        if values.ndim == 2:
            values = values[:, np.newaxis, :]
        if values.ndim != 3:
            raise ValueError("X must be (n_series, l_series) or (n_series, n_channels, l_series)")
        self.bank_ = generate_bank(
            values.shape[2], values.shape[1], self.num_kernels,
            GenOptions(center_weights=self.center_weights, seed=self.seed),
        )
        device_bank(self.bank_, self.device)  # lay the bank out on the GPU once
        return self

    def transform(self, X):
        if self.bank_ is None:
            raise RuntimeError("call fit() before transform()")
        values = np.asarray(getattr(X, "values", X))
        if values.ndim == 2:
            values = values[:, np.newaxis, :]
        return transform(values, self.bank_, self.limits, mode=self.mode, device=self.device).values

    def fit_transform(self, X, y=None):
        return self.fit(X, y).transform(X)
