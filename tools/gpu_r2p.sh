#!/bin/bash
set -x
O=gpurun_out/r2p
mkdir -p $O
for m in opt-13b opt-1.3b opt-30b-tp8; do timeout 300 python tools/cublas_ref.py $m >> $O/cublas.ndjson 2>&1; done
