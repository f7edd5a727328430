# 2-GPU: CTA counts beyond the autotuner's (16..128) candidates — 148 (one per SM) and 296 — for two-shot 1-8 MB and one-shot 256 KB-1 MB
mkdir -p gpurun_out/r40
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for rep in 1 2; do
for b in 128 148 296; do
  timeout 300 $RB launch --world 2 --impl nvrar --algo twoshot --blocks $b --sizes 1048576,2097152,4194304,8388608 --steps 15 > gpurun_out/r40/w2_twoshot_b${b}_rep$rep.jsonl 2>/dev/null; echo "w2 twoshot b$b rc=$?"
  timeout 300 $RB launch --world 2 --impl nvrar --algo oneshot --blocks $b --sizes 262144,524288,1048576 --steps 15 > gpurun_out/r40/w2_oneshot_b${b}_rep$rep.jsonl 2>/dev/null; echo "w2 oneshot b$b rc=$?"
done
done
