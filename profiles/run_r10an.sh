#!/bin/bash
out=gpurun_out/r10an; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "opaque" -q -p no:cacheprovider > $out/pytest.log 2>&1; tail -15 $out/pytest.log
