# 4-GPU: per-thread call-number read vs the barrier broadcast (NVRAR_FLAGS=8), P=1/2/4; quick GPU parity
mkdir -p gpurun_out/r19
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for rep in 1 2; do
for w in 1 2 4; do
  for f in 8 0; do
    NVRAR_FLAGS=$f timeout 300 $RB launch --world $w --impl nvrar --algo oneshot --sizes 65536,131072,524288,1048576 --steps 15 > gpurun_out/r19/w${w}_f${f}_rep$rep.jsonl 2>/dev/null; echo "w$w f$f rep$rep rc=$?"
  done
done
done
for f in 8 0; do
  NVRAR_FLAGS=$f timeout 300 $RB launch --world 4 --impl nvrar --algo hier --sizes 1048576,2097152 --steps 15 > gpurun_out/r19/w4_hier_f${f}.jsonl 2>/dev/null; echo "w4 hier f$f rc=$?"
done
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_timesliced.py tests/test_fuzz.py > gpurun_out/r19/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r19/pytest.log
