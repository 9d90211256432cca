"""BASELINE config 1 on the GPU: FordA-shaped synthetic labelled set
(3,601 series x L=500, 10k kernels) -> transform -> ridge fit + predict,
features kept in HBM; times each stage with CUDA events and compares with
the reference CPU pipeline timings measured in SURVEY.md §6."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2601_17091_b200 import GenOptions, device_bank, generate_bank, ridge, synth_two_class

ds = synth_two_class(1801, 500, seed=1)
values, labels = ds.values[:3601], ds.labels[:3601]
bank = generate_bank(500, 1, 10000, GenOptions(seed=0))
db = device_bank(bank, 0)
x = torch.from_numpy(values).cuda()
feats = torch.empty((x.shape[0], 2 * bank.count), device="cuda")
s = torch.cuda.current_stream().cuda_stream
out = {}
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    db.transform_into(x.data_ptr(), x.shape[0], feats.data_ptr(), feats.shape[1], mode="fast", stream=s)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    model = ridge.fit(feats, labels, alpha=1.0)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    pred = ridge.predict(model, feats)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    out = {"transform_ms": 1e3 * (t1 - t0), "ridge_fit_ms": 1e3 * (t2 - t1), "predict_ms": 1e3 * (t3 - t2),
           "train_accuracy": ridge.accuracy(pred, labels), "series": int(x.shape[0]), "features": int(feats.shape[1])}
out["reference_cpu_survey"] = {"transform_s": 52.5, "ridge_fit_s": 3.4, "host": "8-core Xeon (survey container)"}
print(json.dumps(out))
