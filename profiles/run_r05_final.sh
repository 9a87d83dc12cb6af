#!/bin/bash
# end-of-round check on a fresh box: full GPU suite, smoke(), bench line
out=gpurun_out/r05f; mkdir -p $out
timeout 900 python -m pytest tests -q -m gpu > $out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py > $out/smoke.log 2>&1
timeout 600 python bench.py > $out/bench.log 2>&1
tail -1 $out/bench.log > $out/bench.json
