# 4-GPU: branch-hint + 32-bit-index build vs r19; P=1 instruction-cache counters
mkdir -p gpurun_out/r20
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for w in 1 2 4; do
  timeout 300 $RB launch --world $w --impl nvrar --algo oneshot --sizes 65536,131072,524288,1048576 --steps 15 > gpurun_out/r20/w${w}.jsonl 2>/dev/null; echo "w$w rc=$?"
done
timeout 300 $RB launch --world 4 --impl nvrar --algo hier --sizes 1048576,2097152 --steps 15 > gpurun_out/r20/w4_hier.jsonl 2>/dev/null; echo "w4 hier rc=$?"
M=gpu__time_duration.sum,sm__icc_requests.sum,sm__icc_requests_lookup_miss.sum,sm__icc_requests_lookup_miss_tag_miss.sum,smsp__inst_executed.sum,smsp__warps_issue_stalled_no_instruction.sum,smsp__warps_issue_stalled_long_scoreboard.sum,smsp__warps_issue_stalled_barrier.sum
CUDA_VISIBLE_DEVICES=0 timeout 300 ncu --cache-control none --clock-control none -k regex:flat_kernel --launch-skip 5 --launch-count 3 --metrics $M --csv --log-file gpurun_out/r20/icc.csv python -m paper_2511_09557_b200.profile_emu --solo --algo oneshot --dtype bf16 --bytes 131072 --calls 10 > gpurun_out/r20/icc.out 2>&1; echo "icc rc=$?"
