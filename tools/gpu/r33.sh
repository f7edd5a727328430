# 2-GPU: call number read before griddepcontrol.wait (NVRAR_FLAGS=32) vs default, P=1/2, + a stress run under the flag
mkdir -p gpurun_out/r33
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for rep in 1 2; do
for w in 1 2; do
  for f in 0 32; do
    NVRAR_FLAGS=$f timeout 300 $RB launch --world $w --impl nvrar --algo oneshot --sizes 65536,131072,524288,1048576 --steps 15 > gpurun_out/r33/w${w}_f${f}_rep$rep.jsonl 2>gpurun_out/r33/w${w}_f${f}_rep$rep.err; echo "w$w f$f rep$rep rc=$?"
  done
done
for f in 0 32; do
  NVRAR_FLAGS=$f timeout 300 $RB launch --world 2 --impl nvrar --algo auto --sizes 2097152,8388608 --steps 15 > gpurun_out/r33/w2_auto_f${f}_rep$rep.jsonl 2>/dev/null; echo "w2 auto f$f rc=$?"
done
done
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NVRAR_FLAGS=32 timeout 600 $TR --nproc-per-node 2 --master-port 29661 tests/mp_stress.py --calls 2000 --multicast --registered --sync-every 7 > gpurun_out/r33/stress_p2_f32.log 2>&1; echo "stress f32 rc=$?"; grep -c "OK after" gpurun_out/r33/stress_p2_f32.log
NVRAR_FLAGS=32 timeout 600 python -m pytest tests/test_multigpu.py -x -q -m gpu > gpurun_out/r33/multigpu_f32.txt 2>&1; echo "multigpu f32 rc=$?"
