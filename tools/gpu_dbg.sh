#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_lm.py -q -s -rA > gpurun_out/pytest_cfg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cfg.log
