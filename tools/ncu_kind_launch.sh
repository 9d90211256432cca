#!/bin/bash
# ncu --set full capture of the longest launch of one chunk kind (nck) in the
# measured transform: tools/ncu_kind_launch.sh <tag> <nck> <profile_transform.py args...>
set -u
tag=$1; nck=$2; shift 2
mkdir -p gpurun_out/ncu
RK_PROFILE=1 python tools/profile_transform.py "$@" > gpurun_out/ncu/$tag.plain.log 2> gpurun_out/ncu/$tag.prof.txt || exit 1
skip=$(python - "$tag" "$nck" <<'PY'
import re, sys
lines = [l for l in open(f"gpurun_out/ncu/{sys.argv[1]}.prof.txt") if l.startswith("RK_PROFILE wide")]
per = len(lines) // 2
best, idx = -1, per
for i, l in enumerate(lines[per:]):
    d = dict(kv.split("=") for kv in l.split()[2:])
    if d["nck"] == sys.argv[2] and float(d["ms"]) > best:
        best, idx = float(d["ms"]), per + i
print(idx)
PY
)
echo "tag=$tag nck=$nck skip=$skip" >> gpurun_out/ncu/$tag.plain.log
ncu --set full --clock-control none --import-source on -k regex:rocket_wide_kernel -s $skip -c 1 \
    -o gpurun_out/ncu/$tag python tools/profile_transform.py "$@" > gpurun_out/ncu/$tag.ncu.log 2>&1
