# 2-GPU final check on the last build: GPU suite, smoke, bench N=2 and its reference arm (the driver's scaling-run command)
mkdir -p gpurun_out/r39
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r39/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/r39/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r39/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29671 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r39/bench_n2.json 2> gpurun_out/r39/bench_n2.err; echo "n2 rc=$?"
timeout 600 $TR --nproc-per-node 2 --master-port 29672 bench.py --gpus 2 --impl reference --steps 10 --warmup 3 > gpurun_out/r39/bench_ref_n2.json 2> gpurun_out/r39/bench_ref_n2.err; echo "ref n2 rc=$?"
