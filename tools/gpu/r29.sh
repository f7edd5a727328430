# 4-GPU: final bench lines N=2 and N=4 (+ reference arms), TP=4 decode on the final build
mkdir -p gpurun_out/r29
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29641 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r29/bench_n2.json 2> gpurun_out/r29/bench_n2.err; echo "n2 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29642 bench.py --gpus 2 --impl reference --steps 10 --warmup 3 > gpurun_out/r29/bench_ref_n2.json 2> gpurun_out/r29/bench_ref_n2.err; echo "ref n2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29643 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r29/bench_n4.json 2> gpurun_out/r29/bench_n4.err; echo "n4 rc=$?"
timeout 600 $TR --nproc-per-node 4 --master-port 29644 bench.py --gpus 4 --impl reference --steps 10 --warmup 3 > gpurun_out/r29/bench_ref_n4.json 2> gpurun_out/r29/bench_ref_n4.err; echo "ref n4 rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29645 -m paper_2511_09557_b200.tp_decode --model 70b > gpurun_out/r29/tp_decode_70b_p4.jsonl 2> gpurun_out/r29/tp_decode.err; echo "tp70 rc=$?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29646 -m paper_2511_09557_b200.tp_decode --model 405b --batch 4,16,64 > gpurun_out/r29/tp_decode_405b_p4.jsonl 2> gpurun_out/r29/tp_decode405.err; echo "tp405 rc=$?"
