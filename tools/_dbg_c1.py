import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from bench import CONFIGS, config1_data
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, transform
from oracle.oracle import oracle_transform
cfg = CONFIGS["config1"]
values, labels = config1_data(cfg)
bank = generate_bank(500, 1, 10000, GenOptions(seed=0))
db = device_bank(bank, 0)
x = torch.from_numpy(values).cuda()
for mode in ("fast", "exact"):
    f = torch.empty((len(labels), 20000), device="cuda")
    db.transform_into(x.data_ptr(), len(labels), f.data_ptr(), 20000, mode=mode, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    a = f.cpu().numpy()
    bad = ~np.isfinite(a)
    print(mode, "nonfinite", bad.sum(), "rows", np.unique(np.nonzero(bad)[0])[:10], "cols", np.unique(np.nonzero(bad)[1])[:10])
    if bad.any():
        r = np.nonzero(bad)[0][0]; c = np.nonzero(bad)[1][0]
        ref = oracle_transform(values[r:r+1], bank)
        print("row", r, "col", c, "gpu", a[r, c], "ref", ref[0, c], "kernel", c//2, "d", bank.dilations[c//2], "len", bank.lengths[c//2], "pad", bank.paddings[c//2])
print("values finite", np.isfinite(values).all(), values.shape, values.dtype, np.abs(values).max())
