#!/bin/bash
O=gpurun_out/g5; mkdir -p $O
timeout 900 python tools/gemm_tune.py grid > $O/tune.txt 2>&1
