cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CASCADE_DENSE_PF=4 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_pf4.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_pf4.txt
ARMS="base:X=1;pf2:CASCADE_DENSE_PF=2;pf4:CASCADE_DENSE_PF=4;pf8:CASCADE_DENSE_PF=8" REPS=2 TAG=pf_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="base:X=1;pf2:CASCADE_DENSE_PF=2;pf4:CASCADE_DENSE_PF=4;pf8:CASCADE_DENSE_PF=8" REPS=1 TAG=pf_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
CASCADE_DENSE_PF=4 timeout 600 python scripts/cta_timeline.py mixtral 0,8 pf4 > gpurun_out/tl_mixtral_pf4.txt 2>&1
CASCADE_DENSE_PF=4 timeout 600 python scripts/cta_timeline.py olmoe 0 pf4 > gpurun_out/tl_olmoe_pf4.txt 2>&1
