#!/bin/bash
# ncu --set full capture of the longest wide-kernel launch of one transform.
#   tools/ncu_top_launch.sh <tag> <profile_transform.py args...>
# Runs the transform once with RK_PROFILE=1 (per-launch event times), picks
# the longest launch of the measured (last) transform, then captures it.
set -u
tag=$1; shift
mkdir -p gpurun_out/ncu
RK_PROFILE=1 python tools/profile_transform.py "$@" > gpurun_out/ncu/$tag.plain.log 2> gpurun_out/ncu/$tag.prof.txt || exit 1
skip=$(python - "$tag" <<'PY'
import re, sys
lines = [l for l in open(f"gpurun_out/ncu/{sys.argv[1]}.prof.txt") if l.startswith("RK_PROFILE wide")]
ms = [float(re.search(r"ms=([0-9.]+)", l).group(1)) for l in lines]
n = len(ms)
# two transforms (warm-up 1): the last half is the measured one
per = n // 2
last = ms[per:]
print(per + max(range(len(last)), key=lambda i: last[i]))
PY
)
echo "tag=$tag skip=$skip" >> gpurun_out/ncu/$tag.plain.log
ncu --set full --clock-control none --import-source on -k regex:rocket_wide_kernel -s $skip -c 1 \
    -o gpurun_out/ncu/$tag python tools/profile_transform.py "$@" > gpurun_out/ncu/$tag.ncu.log 2>&1
