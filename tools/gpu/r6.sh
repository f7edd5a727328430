# 1-GPU: PCIe probe, N=1 direct grid sweep, range-replay DRAM traffic, sanitizers, full gpu tests
mkdir -p gpurun_out/r6
cd $GRAFT_REPO_ROOT
timeout 120 python tools/pcie_probe.py > gpurun_out/r6/pcie.json 2>&1; echo "pcie rc=$?"
for u in 1 2 4; do
  NVRAR_DIRECT_UPT=$u timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep > gpurun_out/r6/bench_n1_upt$u.json 2> gpurun_out/r6/bench_n1_upt$u.err; echo "bench upt=$u rc=$?"
done
for h in 4 8 16; do
  NVRAR_HOST_UPT=$h timeout 300 python bench.py --steps 10 --warmup 3 --no-sweep > gpurun_out/r6/bench_n1_hupt$h.json 2> /dev/null; echo "bench hupt=$h rc=$?"
done
timeout 300 ncu --replay-mode range --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r6/ncu_range_direct.csv python -m paper_2511_09557_b200.profile_emu --range --algo auto --dtype f32 --bytes 1048576 > gpurun_out/r6/ncu_range.out 2>&1; echo "ncu range rc=$?"
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tests/sanitize_emu.py > gpurun_out/r6/sanitize_memcheck.txt 2>&1; echo "memcheck rc=$?"
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tests/sanitize_emu.py > gpurun_out/r6/sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?"
timeout 600 compute-sanitizer --tool synccheck --error-exitcode 9 python tests/sanitize_emu.py > gpurun_out/r6/sanitize_synccheck.txt 2>&1; echo "synccheck rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/r6/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r6/pytest_gpu.log
