#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02f
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pack.py tests/test_gpu_parity.py tests/test_gpu_nccl.py -q --timeout 800 -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
timeout 900 python tools/remap_timeline.py --n 30 --G 8 > $OUT/timeline30_G8.json 2> $OUT/timeline.err; echo "timeline rc=$?" >> $OUT/timeline.err
timeout 900 python tools/remap_timeline.py --n 30 --G 2 > $OUT/timeline30_G2.json 2>> $OUT/timeline.err; echo "timeline rc=$?" >> $OUT/timeline.err
