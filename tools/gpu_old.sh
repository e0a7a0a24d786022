#!/bin/bash
cd old_ae6
for i in 1 2 3 4; do timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider 2>&1 | grep -E "first timeout|passed|failed" | head -2; done
