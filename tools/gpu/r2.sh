mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 60 ncu --metrics gpu__time_duration.sum python -c "import os,json; print(json.dumps(dict(os.environ)))" > gpurun_out/ncu_env.log 2>&1
timeout 60 python -c "import os,json; print(json.dumps(dict(os.environ)))" > gpurun_out/plain_env.log 2>&1
NVRAR_SMOKE_KEEP_ENV=1 timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_smoke_keep.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu_keep.log 2>&1; echo "smoke-ncu-keep rc=$?"
