#!/bin/bash
# One GPU iteration: the whole -m gpu suite, then device timings of the named configs.
#   bash tools/gpu_check.sh <outdir> cfg5 cfg2 ...
set -u
O=$1; shift
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python tools/quick_time.py "$@" > $O/quick.log 2>&1; cat $O/quick.log
