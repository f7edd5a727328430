# 4-GPU: reduce-loop batching — perf (two-shot large, one-shot small) + the GPU suites
mkdir -p gpurun_out/r31
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for w in 2 4; do
  timeout 300 $RB launch --world $w --impl nvrar --algo twoshot --sizes 1048576,2097152,4194304,8388608 --steps 15 > gpurun_out/r31/w${w}_twoshot.jsonl 2>/dev/null; echo "w$w twoshot rc=$?"
  timeout 300 $RB launch --world $w --impl nvrar --algo oneshot --sizes 65536,131072,524288,1048576 --steps 15 > gpurun_out/r31/w${w}_oneshot.jsonl 2>/dev/null; echo "w$w oneshot rc=$?"
done
timeout 2000 python -m pytest -q tests -m gpu > gpurun_out/r31/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r31/pytest.log
