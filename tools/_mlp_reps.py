"""Per-rep times of the config-3 TinyMlp transform (tcgen05), to look at run-to-run spread."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import paper_2309_12543_b200 as L

    grid = L.EnvGrid(1.28, 0.01)
    window = L.WindowGeometry.build(0.64, grid)
    V = window.n_masked
    B = 3000
    Rall = L.sample_rotations(np.random.default_rng(0), B)
    Rd = torch.from_numpy(Rall.reshape(B, 9)).cuda()
    model = L.TinyMlp.initial(V, hidden=32, seed=0)
    Y = torch.empty((B, (3 * V + 31) // 32 * 32), dtype=torch.float32, device="cuda")[:, :3 * V]
    for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        model.predict_device(Rd, use_tensor_cores=True, out=Y)
        b.record()
        b.synchronize()
        print(f"rep {k}: {a.elapsed_time(b):.2f} ms")


if __name__ == "__main__":
    main()
