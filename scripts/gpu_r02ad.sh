#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02ad
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_dm.py -q --timeout 600 -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
