# CUDA-core (FMA) vs mma.sync expert FFN at T = 1: GPU tests on the FMA engine, same-call bench A/B, ncu --set full of one FFN launch each.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CASCADE_FFN_FMA=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_fma.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_fma.txt
ARMS="mma:X=1;fma:CASCADE_FFN_FMA=1" REPS=2 TAG=fma_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="mma:X=1;fma:CASCADE_FFN_FMA=1" REPS=2 TAG=fma_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
for arm in mma fma; do
  if [ $arm = fma ]; then export CASCADE_FFN_FMA=1; else unset CASCADE_FFN_FMA; fi
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:expert_ffn -c 2 -o gpurun_out/ffn_t1_$arm python scripts/profile_step.py --ks 0 --layers 2 > gpurun_out/prof_ffn_t1_$arm.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/prof_ffn_t1_$arm.log
done
unset CASCADE_FFN_FMA
