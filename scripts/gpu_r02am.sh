#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02am
mkdir -p $OUT
python tools/proj_probe_tmp.py > $OUT/p.json 2>&1
python tools/stateops_timing.py 32 > $OUT/ops.json 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
