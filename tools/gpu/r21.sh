# 1-GPU: fixed-cost ablations of the one-shot kernel at P=1 (experiment builds from tools/ablate.sh)
mkdir -p gpurun_out/r21
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench launch --world 1 --impl nvrar --algo oneshot --sizes 65536,131072,1048576 --steps 15"
timeout 200 $RB > gpurun_out/r21/base.jsonl 2>/dev/null; echo "base rc=$?"
NVRAR_PDL=0 timeout 200 $RB > gpurun_out/r21/nopdl.jsonl 2>/dev/null; echo "nopdl rc=$?"
NVRAR_FLAGS=2 timeout 200 $RB > gpurun_out/r21/lazy.jsonl 2>/dev/null; echo "lazy rc=$?"
for v in NO_SEQ NO_END NO_SYNC2; do
  NVRAR_LIB=$GRAFT_REPO_ROOT/build_exp/$v/libnvrar_b200.so timeout 200 $RB > gpurun_out/r21/$v.jsonl 2>/dev/null; echo "$v rc=$?"
done
