# 1-GPU, the driver's sequence on the final commit: GPU suite, smoke, bench N=1 and the reference arm
mkdir -p gpurun_out/r48
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r48/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/r48/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r48/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r48/bench_ref_n1.json 2> gpurun_out/r48/bench_ref_n1.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r48/bench_n1.json 2> gpurun_out/r48/bench_n1.err; echo "bench rc=$?"
