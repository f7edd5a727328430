# 4-GPU: long mixed-call stress on the final build (every call kind incl. registered, schedule/CTA/dtype/size switching), with and without delay injection; virtual-rank stress with the dirty-slot invariant
mkdir -p gpurun_out/r30
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes 1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29651 tests/mp_stress.py --calls 4000 --multicast --registered --sync-every 7 > gpurun_out/r30/stress_p2.log 2>&1; echo "p2 rc=$?"; grep -c "OK after" gpurun_out/r30/stress_p2.log
timeout 900 $TR --nproc-per-node 4 --master-port 29652 tests/mp_stress.py --calls 3000 --multicast --registered --sync-every 11 > gpurun_out/r30/stress_p4.log 2>&1; echo "p4 rc=$?"; grep -c "OK after" gpurun_out/r30/stress_p4.log
timeout 900 $TR --nproc-per-node 4 --master-port 29653 tests/mp_stress.py --calls 1500 --registered --jitter 2000 --sync-every 5 > gpurun_out/r30/stress_p4_jitter.log 2>&1; echo "p4 jitter rc=$?"; grep -c "OK after" gpurun_out/r30/stress_p4_jitter.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python tests/stress_emu.py --calls 3000 --nodes 2 --gpus 4 --check-dirty > gpurun_out/r30/stress_emu_2x4.log 2>&1; echo "emu rc=$?"; tail -1 gpurun_out/r30/stress_emu_2x4.log
