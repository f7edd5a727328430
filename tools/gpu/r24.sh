# 4-GPU: counter write-back mid-kernel (flat) — P=1/2/4 one-shot + two-shot; parity suites
mkdir -p gpurun_out/r24
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for w in 1 2 4; do
  timeout 300 $RB launch --world $w --impl nvrar --algo oneshot --sizes 65536,131072,524288,1048576 --steps 15 > gpurun_out/r24/w${w}.jsonl 2>/dev/null; echo "w$w rc=$?"
done
timeout 300 $RB launch --world 4 --impl nvrar --algo twoshot --sizes 1048576,2097152,4194304 --steps 15 > gpurun_out/r24/w4_twoshot.jsonl 2>/dev/null; echo "w4 twoshot rc=$?"
timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_phases.py tests/test_timesliced.py tests/test_fuzz.py tests/test_multigpu.py > gpurun_out/r24/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r24/pytest.log
