"""Small transforms that reach every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per gpurun call):

* the wide kernel, fast and exact, on a config-2-shaped bank (L=1024) with
  enough series for two-series items and half-warp chunks, staged by 1-D TMA
  bulk copies (aligned input) and by the cooperative copy (unaligned input);
* fast-mode MPV (wide MPV kernels) and exact MPV / float64 (staged cell
  kernels);
* a 3-channel bank (run-time slot loop) and a series too long for shared
  memory (GMEM variants, unstaged float64 cell kernel);
* the pinned-host pipeline and the pageable ring.

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_slice.py
Every result is checked against the oracle so a run that "passes" the
sanitizer also computed the right features."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.oracle import oracle_transform  # noqa: E402
from oracle.parity import check_fast  # noqa: E402
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, synth_random, transform  # noqa: E402

small = "--small" in sys.argv  # racecheck: fewer series (its shared-memory tracking is slow)


def dev_run(bank, values, mode, fpk=2, precision="single", offset=0):
    db = device_bank(bank, 0)
    dt = torch.float64 if precision == "double" else torch.float32
    flat = torch.zeros(values.size + offset, dtype=dt)
    flat[offset:] = torch.from_numpy(values.astype(np.float64 if precision == "double" else np.float32).ravel())
    xd = flat.cuda()
    out = torch.empty((values.shape[0], bank.count * fpk), device="cuda", dtype=dt)
    db.transform_into(xd.data_ptr() + offset * xd.element_size(), values.shape[0], out.data_ptr(), out.shape[1],
                      mode=mode, fpk=fpk, precision=precision)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def main():
    n = 1200 if small else 6000
    rows = np.arange(0, n, n // 12)
    bank = generate_bank(1024, 1, 1000, GenOptions(seed=0))
    info = device_bank(bank, 0).info
    assert info["n_half_chunks"] + info["n_quarter_chunks"] + info["n_eighth_chunks"] > 0
    values = synth_random(n, 1, 1024, seed=1).values
    ref = oracle_transform(values[rows], bank)
    assert dev_run(bank, values, "exact")[rows].tobytes() == ref.tobytes()
    check_fast(dev_run(bank, values, "fast")[rows], ref, values[rows], bank)
    assert dev_run(bank, values, "exact", offset=1)[rows].tobytes() == ref.tobytes()  # cooperative staging
    ref3 = oracle_transform(values[rows], bank, include_mpv=True)
    check_fast(dev_run(bank, values, "fast", fpk=3)[rows], ref3, values[rows], bank, fpk=3)
    m = values[:64]
    assert dev_run(bank, m, "exact", fpk=3).tobytes() == oracle_transform(m, bank, include_mpv=True).tobytes()
    assert dev_run(bank, m, "exact", precision="double").tobytes() == \
        oracle_transform(m, bank, precision="double").tobytes()
    # pinned-host pipeline and pageable ring
    xp = torch.from_numpy(values).pin_memory()
    op = torch.empty((n, bank.count * 2)).pin_memory()
    device_bank(bank, 0).transform_into(xp.data_ptr(), n, op.data_ptr(), bank.count * 2, mode="exact")
    assert op.numpy()[rows].tobytes() == ref.tobytes()
    assert transform(values, bank, mode="exact").values[rows].tobytes() == ref.tobytes()
    # 3 channels (run-time slot loop)
    b3 = generate_bank(512, 3, 600, GenOptions(seed=2))
    v3 = synth_random(800 if not small else 200, 3, 512, seed=3).values
    r3 = oracle_transform(v3[:16], b3)
    assert dev_run(b3, v3, "exact")[:16].tobytes() == r3.tobytes()
    check_fast(dev_run(b3, v3, "fast")[:16], r3, v3[:16], b3)
    # series longer than shared memory: GMEM wide kernels, unstaged float64 cell kernel
    bl = generate_bank(70_000, 1, 40, GenOptions(seed=4))
    vl = synth_random(3, 1, 70_000, seed=5).values
    rl = oracle_transform(vl, bl)
    assert dev_run(bl, vl, "exact").tobytes() == rl.tobytes()
    check_fast(dev_run(bl, vl, "fast"), rl, vl, bl)
    assert dev_run(bl, vl[:1], "exact", precision="double").tobytes() == \
        oracle_transform(vl[:1], bl, precision="double").tobytes()
    print("sanitize slice ok")


if __name__ == "__main__":
    main()
