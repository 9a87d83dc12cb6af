#!/bin/bash
out=gpurun_out/r10aq; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "misses_nothing" -q -p no:cacheprovider > $out/pytest.log 2>&1; tail -5 $out/pytest.log
