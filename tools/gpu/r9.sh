# 4-GPU: multigpu tests (incl. 8 ranks on 4 GPUs), bench N=4, timeline, NVLink/stall captures, TP decode, NCCL best-of
mkdir -p gpurun_out/r9
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q tests/test_multigpu.py --durations=30 > gpurun_out/r9/pytest_multigpu_4gpu.log 2>&1; echo "multigpu tests rc=$?"
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r9/bench_n4.json 2> gpurun_out/r9/bench_n4.err; echo "bench n4 rc=$?"
timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 -m paper_2511_09557_b200.timeline --bytes 131072 --algo oneshot --blocks 64 > gpurun_out/r9/timeline_p4_128k.json 2> gpurun_out/r9/timeline.err; echo "timeline rc=$?"
NVLP="python -m paper_2511_09557_b200.nvlprofile --world 4 --timeout 5 --calls 3"
STALL=smsp__warps_issue_stalled_long_scoreboard.sum,smsp__warps_issue_stalled_sleeping.sum,smsp__warps_issue_stalled_barrier.sum,smsp__warps_issue_stalled_lg_throttle.sum,smsp__warps_issue_stalled_membar.sum,smsp__warps_issue_stalled_wait.sum,smsp__warps_issue_stalled_no_instruction.sum,smsp__warps_issue_stalled_drain.sum,smsp__warps_issue_stalled_branch_resolving.sum,smsp__warps_issue_stalled_selected.sum,smsp__warps_issue_stalled_short_scoreboard.sum,smsp__warps_issue_stalled_mio_throttle.sum
for algo in oneshot twoshot hier; do
  for size in 131072 1048576 2097152; do
    timeout 120 ncu --devices 0 -k regex:"flat_kernel|hier_kernel" --launch-skip 2 --launch-count 1 --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum --csv --log-file gpurun_out/r9/nvl_${algo}_${size}.csv $NVLP --algos $algo --sizes $size > gpurun_out/r9/nvl_${algo}_${size}.out 2>&1; echo "nvl $algo $size rc=$?"
    timeout 120 ncu --devices 0 -k regex:"flat_kernel|hier_kernel" --launch-skip 2 --launch-count 1 --metrics gpu__time_duration.sum,smsp__cycles_active.sum,$STALL --csv --log-file gpurun_out/r9/stall_${algo}_${size}.csv $NVLP --algos $algo --sizes $size > gpurun_out/r9/stall_${algo}_${size}.out 2>&1; echo "stall $algo $size rc=$?"
  done
done
timeout 1200 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29583 -m paper_2511_09557_b200.tp_decode --model 70b > gpurun_out/r9/tp_decode_70b_p4.jsonl 2> gpurun_out/r9/tp_decode.err; echo "tp decode rc=$?"
timeout 2700 python -m paper_2511_09557_b200.rankbench nccl-best --world 4 > gpurun_out/r9/nccl_best_p4.jsonl 2> gpurun_out/r9/nccl_best.err; echo "nccl best rc=$?"
