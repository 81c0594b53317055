cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu4.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_r01.csv python scripts/profile_step.py --ks 0,8 > gpurun_out/prof_launch.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/prof_launch.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:stream_gemv_kernel -s 5 -c 6 -o gpurun_out/gemv_full_r01 python scripts/profile_step.py --ks 8 --layers 2 > gpurun_out/prof_full.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/prof_full.log
