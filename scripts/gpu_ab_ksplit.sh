# Key-split attention chunk tiles (4 warps share a 16-row tile): bitwise check, tests, A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_shapes.py -x -q -k key_split > gpurun_out/pytest_ksplit_bitwise.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_ksplit_bitwise.txt
if [ $rc -ne 0 ]; then exit 0; fi
ARMS="ksplit:CASCADE_ATTN_KSPLIT=1;base:X=1" REPS=3 TAG=ksplit4_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="ksplit:CASCADE_ATTN_KSPLIT=1;base:X=1" REPS=1 TAG=ksplit4_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
CASCADE_ATTN_KSPLIT=1 timeout 600 python scripts/cta_timeline.py mixtral 4 ksplit > gpurun_out/tl_mixtral_k4_ksplit.txt 2>&1
