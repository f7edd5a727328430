# 2-GPU: N>1 host-buffer e2e per schedule vs the host CTA cap (NVRAR_HOST_CTAS), P=2
mkdir -p gpurun_out/r45
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29700
for c in 8 16 32 64 128; do
  for b in 262144 1048576 4194304; do
    port=$((port+1))
    NVRAR_HOST_CTAS=$c timeout 300 $TR --master-port $port tools/e2e_probe_mp.py --bytes $b >> gpurun_out/r45/e2e.txt 2>>gpurun_out/r45/e2e.err; echo "c$c b$b rc=$?"
  done
done
