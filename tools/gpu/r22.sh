# 4-GPU: call-counter write-back early (NVRAR_FLAGS=1) / lazy length check (2) / both (3) vs default, P=1/2/4, current build
mkdir -p gpurun_out/r22
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for rep in 1 2; do
for w in 1 2 4; do
  for f in 0 1 2 3; do
    NVRAR_FLAGS=$f timeout 300 $RB launch --world $w --impl nvrar --algo oneshot --sizes 65536,131072,524288,1048576 --steps 15 > gpurun_out/r22/w${w}_f${f}_rep$rep.jsonl 2>/dev/null; echo "w$w f$f rep$rep rc=$?"
  done
done
done
for f in 0 1; do
  NVRAR_FLAGS=$f timeout 300 $RB launch --world 4 --impl nvrar --algo hier --sizes 1048576,2097152 --steps 15 > gpurun_out/r22/w4_hier_f$f.jsonl 2>/dev/null; echo "w4 hier f$f rc=$?"
done
