# 1-GPU: N=1 direct schedule — 256-byte L2 fetch hint on device inputs (NVRAR_DEV_L2FETCH=1) A/B, interleaved
mkdir -p gpurun_out/r46
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  for f in 0 1; do
    NVRAR_DEV_L2FETCH=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/r46/n1_l2f${f}_$rep.json 2>/dev/null; echo "f$f rep$rep rc=$?"
  done
done
