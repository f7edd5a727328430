# 2-GPU: one-shot specialisation A/B, N=1 direct CTA sweep
mkdir -p gpurun_out/r10
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for rep in 1 2; do
for f in 0 1; do
  NVRAR_FAST_ONESHOT=$f timeout 400 $RB launch --world 2 --impl nvrar --algo oneshot --sizes 65536,131072,262144,524288,1048576 > gpurun_out/r10/fast${f}_rep$rep.jsonl 2> gpurun_out/r10/fast${f}_rep$rep.err; echo "fast $f rc=$?"
done
done
for f in 0 1; do
  NVRAR_FAST_ONESHOT=$f timeout 400 $RB launch --world 2 --impl nvrar --algo oneshot --producer gemm --sizes 131072,1048576 > gpurun_out/r10/fast${f}_prod.jsonl 2> gpurun_out/r10/fast${f}_prod.err; echo "fast $f prod rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 -m paper_2511_09557_b200.timeline --bytes 131072 --algo oneshot --blocks 64 > gpurun_out/r10/timeline_p2_128k_fast.json 2> gpurun_out/r10/timeline.err; echo "timeline rc=$?"
export CUDA_VISIBLE_DEVICES=0
for c in 19 32 37 74; do
  NVRAR_DIRECT_CTAS=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/r10/bench_n1_ctas$c.json 2> gpurun_out/r10/bench_n1_ctas$c.err; echo "bench ctas=$c rc=$?"
done
