# 1-GPU: instruction-cache behaviour of the one-shot kernel at P=1 (specialised vs general), steady state (no cache flush)
mkdir -p gpurun_out/r18
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,sm__icc_requests.sum,sm__icc_requests_lookup_miss.sum,sm__icc_requests_lookup_miss_tag_miss.sum,smsp__inst_executed.sum,smsp__warps_issue_stalled_no_instruction.sum,smsp__warps_issue_stalled_long_scoreboard.sum,smsp__warps_issue_stalled_barrier.sum
for f in 1 0; do
  NVRAR_FAST_ONESHOT=$f timeout 300 ncu --cache-control none --clock-control none -k regex:flat_kernel --launch-skip 5 --launch-count 3 --metrics $M --csv --log-file gpurun_out/r18/icc_fast$f.csv python -m paper_2511_09557_b200.profile_emu --solo --algo oneshot --dtype bf16 --bytes 131072 --calls 10 > gpurun_out/r18/icc_fast$f.out 2>&1; echo "icc fast=$f rc=$?"
done
timeout 300 ncu --cache-control none --clock-control none -k regex:k_main --launch-skip 20 --launch-count 3 --metrics $M --csv --log-file gpurun_out/r18/icc_micro.csv ./tools/launch_micro > gpurun_out/r18/icc_micro.out 2>&1; echo "icc micro rc=$?"
