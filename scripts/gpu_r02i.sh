#!/bin/bash
set -u
export HQ_NO_BUILD=1
OUT=gpurun_out/r02i
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "tests rc=$?" >> $OUT/gputests.log
python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
