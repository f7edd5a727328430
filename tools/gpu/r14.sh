# 1-GPU: where a state-reading kernel's fixed cost goes (launch_micro variants, small/large params); N=1 bench with the new host grid
mkdir -p gpurun_out/r14
cd $GRAFT_REPO_ROOT
LM_VARIANTS=1 timeout 120 ./tools/launch_micro > gpurun_out/r14/launch_micro_variants.txt 2>&1; echo "lm rc=$?"
LM_VARIANTS=1 timeout 120 ./tools/launch_micro_bigparam > gpurun_out/r14/launch_micro_variants_bigparam.txt 2>&1; echo "lm big rc=$?"
for h in 32 64; do
  NVRAR_HOST_UPT=$h timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/r14/bench_n1_h$h.json 2> gpurun_out/r14/bench_n1_h$h.err; echo "bench hupt=$h rc=$?"
done
