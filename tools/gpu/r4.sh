# 2-GPU: NVRAR vs direct NCCL (best over algo x proto x lib), producer mode, NVLink counters
mkdir -p gpurun_out/r4
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
nvidia-smi topo -m > gpurun_out/r4/topo.txt 2>&1
timeout 600 $RB launch --world 2 --impl nvrar > gpurun_out/r4/nvrar.jsonl 2> gpurun_out/r4/nvrar.err; echo "nvrar rc=$?"
timeout 600 $RB launch --world 2 --impl nvrar --producer gemm > gpurun_out/r4/nvrar_prod.jsonl 2> gpurun_out/r4/nvrar_prod.err; echo "nvrar prod rc=$?"
timeout 600 $RB launch --world 2 --impl nccl --nccl-lib torch --producer gemm > gpurun_out/r4/nccl_prod.jsonl 2> gpurun_out/r4/nccl_prod.err; echo "nccl prod rc=$?"
timeout 600 $RB launch --world 2 --impl nccl --nccl-lib system > gpurun_out/r4/nccl_sys_default.jsonl 2> gpurun_out/r4/nccl_sys_default.err; echo "nccl sys rc=$?"
timeout 600 $RB launch --world 2 --impl nvrar --profile --calls 3 --sizes 131072,1048576,2097152 --algo oneshot --show-output \
  --ncu-rank0 "ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:flat_kernel|hier_kernel --csv --log-file gpurun_out/r4/ncu_nvl_oneshot.csv" \
  > gpurun_out/r4/ncu1.out 2> gpurun_out/r4/ncu1.err; echo "ncu rc=$?"
timeout 1800 $RB nccl-best --world 2 > gpurun_out/r4/nccl_best.txt 2> gpurun_out/r4/nccl_best.err; echo "nccl best rc=$?"
