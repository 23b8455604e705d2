"""Golden fixture for TinyMlp training: the REAL reference's train_approximator
on a small window (W = 6, 93 kept points), a short fixed budget.

    python tests/golden/make_training.py      # build container only (/root/reference)
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import linksdf as ref  # noqa: E402  (reference, read-only)

HERE = Path(__file__).resolve().parent
pts = ref.masked_window_points(6)
cfg = ref.TrainingConfig(steps=300, eval_every=100, screen_size=128, val_size=512, target_max_error=1.0, seed=3)
model = ref.train_approximator(pts, cfg)
np.savez_compressed(HERE / "training.npz", points=pts, w1=model.w1, b1=model.b1, w2=model.w2, b2=model.b2,
                    history=np.asarray(model.history, dtype=np.float64),
                    val_max=np.float64(model.validation_max_error), val_mae=np.float64(model.validation_mean_error))
print("saved", pts.shape, model.validation_max_error)
