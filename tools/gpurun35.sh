#!/bin/bash
CPPP_DEBUG_TTM=1 timeout 600 python -m pytest tests/test_gpu_parity.py -k "split_units" -q -s 2>&1 | grep -E "stream-K|passed|failed" | sort | uniq -c | head
