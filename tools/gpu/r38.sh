# 1-GPU (final build, e2e through the C ABI), the driver's sequence: GPU suite, smoke, smoke launch list under ncu, bench N=1 and the reference arm, ncu of the headline kernel
mkdir -p gpurun_out/r38
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r38/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/r38/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r38/smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r38/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r38/smoke_ncu.log 2>&1; echo "smoke ncu rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r38/bench_ref_n1.json 2> gpurun_out/r38/bench_ref_n1.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r38/bench_n1.json 2> gpurun_out/r38/bench_n1.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r38/launches_bench_n1.csv python bench.py --steps 2 --warmup 3 --no-sweep > gpurun_out/r38/bench_ncu.log 2>&1; echo "bench ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:direct_kernel --launch-skip 20 --launch-count 1 -o gpurun_out/r38/direct_n1 python -m paper_2511_09557_b200.profile_emu --algo auto --dtype f32 --bytes 1048576 --calls 30 > gpurun_out/r38/ncu_full.log 2>&1; echo "ncu full rc=$?"
