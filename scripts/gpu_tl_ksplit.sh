cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 0 4; do
CASCADE_ATTN_KSPLIT=1 timeout 600 python scripts/cta_timeline.py mixtral $k ksplit > gpurun_out/tl_mixtral_k${k}_ksplit.txt 2>&1
done
