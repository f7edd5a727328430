# 2-GPU: NVLink TX bytes + stall counters per (schedule, size) on rank 0; N=1 e2e modes; N=1 steady-state DRAM traffic
mkdir -p gpurun_out/r8
cd $GRAFT_REPO_ROOT
NVLP="python -m paper_2511_09557_b200.nvlprofile --world 2 --timeout 5 --calls 3"
STALL=smsp__warps_issue_stalled_long_scoreboard.sum,smsp__warps_issue_stalled_sleeping.sum,smsp__warps_issue_stalled_barrier.sum,smsp__warps_issue_stalled_lg_throttle.sum,smsp__warps_issue_stalled_membar.sum,smsp__warps_issue_stalled_wait.sum,smsp__warps_issue_stalled_no_instruction.sum,smsp__warps_issue_stalled_drain.sum,smsp__warps_issue_stalled_branch_resolving.sum,smsp__warps_issue_stalled_selected.sum,smsp__warps_issue_stalled_short_scoreboard.sum,smsp__warps_issue_stalled_mio_throttle.sum
for algo in oneshot twoshot hier; do
  for size in 131072 524288 1048576 2097152; do
    timeout 120 ncu --devices 0 -k regex:"flat_kernel|hier_kernel" --launch-skip 2 --launch-count 1 --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum --csv --log-file gpurun_out/r8/nvl_${algo}_${size}.csv $NVLP --algos $algo --sizes $size > gpurun_out/r8/nvl_${algo}_${size}.out 2>&1; echo "nvl $algo $size rc=$?"
    timeout 120 ncu --devices 0 -k regex:"flat_kernel|hier_kernel" --launch-skip 2 --launch-count 1 --metrics gpu__time_duration.sum,smsp__cycles_active.sum,$STALL --csv --log-file gpurun_out/r8/stall_${algo}_${size}.csv $NVLP --algos $algo --sizes $size > gpurun_out/r8/stall_${algo}_${size}.out 2>&1; echo "stall $algo $size rc=$?"
  done
done
export CUDA_VISIBLE_DEVICES=0
for m in zerocopy split; do
  for c in 131072 262144 524288; do
    NVRAR_HOST_MODE=$m NVRAR_SPLIT_CHUNK=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-sweep > gpurun_out/r8/bench_n1_${m}_${c}.json 2> gpurun_out/r8/bench_n1_${m}_${c}.err; echo "bench $m $c rc=$?"
    if [ $m = zerocopy ]; then break; fi
  done
done
timeout 300 ncu --cache-control none -k regex:direct_kernel --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r8/ncu_rotate_direct.csv python -m paper_2511_09557_b200.profile_emu --rotate --algo auto --dtype f32 --bytes 1048576 > gpurun_out/r8/ncu_rotate.out 2>&1; echo "ncu rotate rc=$?"
