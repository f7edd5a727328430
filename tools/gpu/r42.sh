# 2-GPU: phase timelines of the P=2 1 MB one-shot (the N=2 headline) and 8 MB two-shot
mkdir -p gpurun_out/r42
cd $GRAFT_REPO_ROOT
TL="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TL --master-port 29681 -m paper_2511_09557_b200.timeline --bytes 1048576 --algo oneshot --blocks 128 > gpurun_out/r42/timeline_p2_1MB_oneshot.json 2> gpurun_out/r42/timeline1.err; echo "timeline 1MB rc=$?"
timeout 300 $TL --master-port 29682 -m paper_2511_09557_b200.timeline --bytes 8388608 --algo twoshot --blocks 128 > gpurun_out/r42/timeline_p2_8MB_twoshot.json 2> gpurun_out/r42/timeline8.err; echo "timeline 8MB rc=$?"
