cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__shared_mem_config_size --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_um.csv python scripts/profile_step.py --ks 0 --layers 4 > gpurun_out/prof_um.log 2>&1
echo "rc=$?" >> gpurun_out/prof_um.log
