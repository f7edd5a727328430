# 4-GPU: full GPU suite at 4 GPUs, bench N=4; on GPU 0: host-input L2 fetch-size A/B for the N=1 e2e, P=1 fixed cost
mkdir -p gpurun_out/r13
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/r13/pytest_gpu_4gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r13/pytest_gpu_4gpu.log
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 4 > gpurun_out/r13/bench_n4.json 2> gpurun_out/r13/bench_n4.err; echo "bench n4 rc=$?"
timeout 300 python -m paper_2511_09557_b200.rankbench launch --world 1 --impl nvrar --sizes 65536,131072,1048576 > gpurun_out/r13/p1.jsonl 2> gpurun_out/r13/p1.err; echo "p1 rc=$?"
export CUDA_VISIBLE_DEVICES=0
for f in 0 1; do
  for h in 8 16 32; do
    NVRAR_HOST_L2FETCH=$f NVRAR_HOST_UPT=$h timeout 300 python bench.py --steps 10 --warmup 3 --no-sweep > gpurun_out/r13/bench_n1_l2f${f}_h$h.json 2> gpurun_out/r13/bench_n1_l2f${f}_h$h.err; echo "bench l2f=$f hupt=$h rc=$?"
  done
done
