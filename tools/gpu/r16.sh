# 2-GPU: CTA shape sweep for the small-message one-shot (threads per CTA x CTAs per rank), P=1 and P=2
mkdir -p gpurun_out/r16
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for w in 1 2; do
  for t in 128 256 512; do
    for b in 8 16 32 64; do
      NVRAR_THREADS=$t timeout 300 $RB launch --world $w --impl nvrar --algo oneshot --blocks $b --sizes 65536,131072,262144 --steps 10 > gpurun_out/r16/w${w}_t${t}_b${b}.jsonl 2>/dev/null; echo "w$w t$t b$b rc=$?"
    done
  done
done
