# 2-GPU: single-process ncu captures of the per-rank kernels (device 0 only), flag A/B, N=1 range traffic
mkdir -p gpurun_out/r7
cd $GRAFT_REPO_ROOT
NVLP="python -m paper_2511_09557_b200.nvlprofile --world 2"
timeout 120 $NVLP --sizes 131072 --algos oneshot > gpurun_out/r7/nvlp_plain.txt 2>&1; echo "nvlp plain rc=$?"
timeout 300 ncu --devices 0 -k regex:"flat_kernel|hier_kernel" --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum --csv --log-file gpurun_out/r7/ncu_nvl.csv $NVLP --timeout 5 > gpurun_out/r7/ncu_nvl.out 2>&1; echo "ncu nvl rc=$?"
timeout 300 ncu --devices 0 -k regex:"flat_kernel|hier_kernel" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r7/ncu_dram.csv $NVLP --timeout 5 > gpurun_out/r7/ncu_dram.out 2>&1; echo "ncu dram rc=$?"
timeout 300 ncu --devices 0 -k regex:"flat_kernel|hier_kernel" --section WarpStateStats --csv --log-file gpurun_out/r7/ncu_warpstate.csv $NVLP --sizes 131072,1048576 --timeout 5 > gpurun_out/r7/ncu_warpstate.out 2>&1; echo "ncu warpstate rc=$?"
timeout 300 ncu --devices 0 -k regex:"flat_kernel" --section SourceCounters --section WarpStateStats --import-source on -o gpurun_out/r7/oneshot_p2_128k $NVLP --sizes 131072 --algos oneshot --timeout 5 > gpurun_out/r7/ncu_source.out 2>&1; echo "ncu source rc=$?"
RB="python -m paper_2511_09557_b200.rankbench"
for f in 0 1 2 3; do
  NVRAR_FLAGS=$f timeout 400 $RB launch --world 2 --impl nvrar --sizes 65536,131072,262144,524288,1048576,2097152 > gpurun_out/r7/flags$f.jsonl 2> gpurun_out/r7/flags$f.err; echo "flags $f rc=$?"
done
for f in 0 3; do
  NVRAR_FLAGS=$f timeout 400 $RB launch --world 2 --impl nvrar --producer gemm --sizes 131072,1048576 > gpurun_out/r7/flags${f}_prod.jsonl 2> gpurun_out/r7/flags${f}_prod.err; echo "flags $f prod rc=$?"
done
CUDA_VISIBLE_DEVICES=0 timeout 300 ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv --log-file gpurun_out/r7/ncu_range_direct.csv python -m paper_2511_09557_b200.profile_emu --range --algo auto --dtype f32 --bytes 1048576 > gpurun_out/r7/ncu_range.out 2>&1; echo "ncu range rc=$?"
