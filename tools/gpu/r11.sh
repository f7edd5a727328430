# 4-GPU: one-shot specialisation A/B at P=2 and P=4 (out-of-line watchdog build), N=1 default grid, hier timeline P=4 1 MB
mkdir -p gpurun_out/r11
cd $GRAFT_REPO_ROOT
RB="python -m paper_2511_09557_b200.rankbench"
for w in 2 4; do
for f in 0 1; do
  NVRAR_FAST_ONESHOT=$f timeout 400 $RB launch --world $w --impl nvrar --algo oneshot --sizes 65536,131072,262144,524288,1048576 > gpurun_out/r11/p${w}_fast$f.jsonl 2> gpurun_out/r11/p${w}_fast$f.err; echo "p$w fast $f rc=$?"
done
timeout 400 $RB launch --world $w --impl nvrar --algo hier --sizes 524288,1048576,2097152 > gpurun_out/r11/p${w}_hier.jsonl 2> gpurun_out/r11/p${w}_hier.err; echo "p$w hier rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 -m paper_2511_09557_b200.timeline --bytes 1048576 --algo hier --blocks 128 > gpurun_out/r11/timeline_p4_1MB_hier.json 2> gpurun_out/r11/timeline.err; echo "timeline rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r11/bench_n1.json 2> gpurun_out/r11/bench_n1.err; echo "bench n1 rc=$?"
