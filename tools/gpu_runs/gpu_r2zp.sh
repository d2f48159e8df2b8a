#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q 2>&1 | grep -v "^\s*$" | grep -A30 "FAILED\|Error\|assert" | head -60
