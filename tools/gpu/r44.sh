# 4-GPU: the whole GPU suite on the final build (multi-GPU tests incl. the 8-rank layouts as 8 processes on 4 GPUs)
mkdir -p gpurun_out/r44
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r44/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/r44/pytest_gpu.log
