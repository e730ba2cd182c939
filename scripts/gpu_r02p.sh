#!/bin/bash
set -u
OUT=gpurun_out/r02p6
mkdir -p $OUT
timeout 600 tools/stream_bench 32 20 8,9,10,20,21,22 > $OUT/stream_a.jsonl 2>&1
