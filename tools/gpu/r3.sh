mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_smoke3.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu3.log 2>&1; echo "smoke-ncu rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; echo "smoke rc=$?"
