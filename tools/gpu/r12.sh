# 2-GPU: full GPU suite (incl. multigpu at P=2), smoke, bench N=1 and N=2 on the current build
mkdir -p gpurun_out/r12
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/r12/pytest_gpu_2gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r12/pytest_gpu_2gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r12/smoke.log 2>&1; echo "smoke rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > gpurun_out/r12/bench_n1.json 2> gpurun_out/r12/bench_n1.err; echo "bench n1 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference > gpurun_out/r12/bench_ref_n1.json 2> gpurun_out/r12/bench_ref_n1.err; echo "bench ref n1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/r12/bench_n2.json 2> gpurun_out/r12/bench_n2.err; echo "bench n2 rc=$?"
