#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TUNE_ARGS=--bf16 bash tools/tune_run.sh > gpurun_out/tune_summary_bf16.txt 2>&1
