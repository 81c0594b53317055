cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:stream_gemv -c 4 -o gpurun_out/gemv_full_$TAG python scripts/profile_step.py --ks ${KS:-8} --layers 2 > gpurun_out/prof_full_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof_full_$TAG.log
