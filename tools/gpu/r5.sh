# 2-GPU: new GPU tests, NCCL direct + best-of, ncu on rank 0, timeline, bench N=2
mkdir -p gpurun_out/r5
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
timeout 900 python -m pytest -x -q tests/test_timesliced.py tests/test_fuzz.py tests/test_binding_gpu.py --durations=15 > gpurun_out/r5/pytest_new.log 2>&1; echo "pytest new rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5/smoke.log 2>&1; echo "smoke rc=$?"
NCCL_DEBUG=INFO timeout 300 $RB launch --world 2 --impl nccl --nccl-lib torch --sizes 131072,1048576 --show-output > gpurun_out/r5/nccl_torch_dbg.jsonl 2> gpurun_out/r5/nccl_torch_dbg.err; echo "nccl dbg rc=$?"
timeout 300 $RB launch --world 2 --impl nvrar --profile --calls 3 --sizes 131072 --algo oneshot --show-output --timeout 240 \
  --ncu-rank0 "ncu --metrics gpu__time_duration.sum -k regex:flat_kernel --csv --log-file gpurun_out/r5/ncu_t.csv" \
  > gpurun_out/r5/ncu_t.out 2> gpurun_out/r5/ncu_t.err; echo "ncu time rc=$?"
timeout 400 $RB launch --world 2 --impl nvrar --profile --calls 3 --sizes 131072,1048576,2097152 --algo oneshot --show-output --timeout 360 \
  --ncu-rank0 "ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:flat_kernel|hier_kernel --csv --log-file gpurun_out/r5/ncu_nvl.csv" \
  > gpurun_out/r5/ncu_nvl.out 2> gpurun_out/r5/ncu_nvl.err; echo "ncu nvl rc=$?"
timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 -m paper_2511_09557_b200.timeline --bytes 131072 --algo oneshot --blocks 64 > gpurun_out/r5/timeline_p2_128k.json 2> gpurun_out/r5/timeline.err; echo "timeline rc=$?"
timeout 600 $RB launch --world 2 --impl nccl --nccl-lib torch --producer gemm > gpurun_out/r5/nccl_prod.jsonl 2> gpurun_out/r5/nccl_prod.err; echo "nccl prod rc=$?"
timeout 2400 $RB nccl-best --world 2 > gpurun_out/r5/nccl_best_p2.jsonl 2> gpurun_out/r5/nccl_best.err; echo "nccl best rc=$?"
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29578 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r5/bench_n2.json 2> gpurun_out/r5/bench_n2.err; echo "bench rc=$?"
