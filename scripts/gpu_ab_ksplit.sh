# Attention tile form per width (CASCADE_ATTN_KSPLIT=3, default) vs key split (1): bitwise check, tests, A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_shapes.py -q -k key_split > gpurun_out/pytest_ksplit_bitwise.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_ksplit_bitwise.txt
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ks3.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gpu_ks3.txt
if [ $rc -ne 0 ]; then exit 0; fi
ARMS="ks3:X=1;ks1:CASCADE_ATTN_KSPLIT=1;ks0:CASCADE_ATTN_KSPLIT=0" REPS=2 TAG=ksplit6_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="ks3:X=1;ks1:CASCADE_ATTN_KSPLIT=1;ks0:CASCADE_ATTN_KSPLIT=0" REPS=2 TAG=ksplit6_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="ks3:X=1;ks1:CASCADE_ATTN_KSPLIT=1;ks0:CASCADE_ATTN_KSPLIT=0" REPS=1 TAG=ksplit6_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
