# Iteration + same-call A/B for the round-2 second-session latency work (attention cluster merge, parallel top-k).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-a1}
CASCADE_DEBUG_CLUSTER=1 timeout 300 python -c "
import paper_2506_20675_b200 as cb
for c in ['tiny','mixtral','olmoe','qwen15']:
    sh = cb.preset(c); m = cb.Model(sh, 1); s = cb.Session(m, max_ctx=1088, k_max=8); print(c, 'ok'); s.close(); m.close()
" > gpurun_out/clusters_$TAG.txt 2>&1
TL_CFGS="${TL_CFGS:-mixtral olmoe}" TAG=$TAG bash scripts/gpu_iter.sh
if [ -z "$NO_AB" ]; then
ARMS="${ARMS:-new:X=1;noattn:CASCADE_ATTN_CLUSTER=0;notopk:CASCADE_TOPK_PAR=0}" REPS=${REPS:-2} TAG=${TAG}_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="${ARMS:-new:X=1;noattn:CASCADE_ATTN_CLUSTER=0;notopk:CASCADE_TOPK_PAR=0}" REPS=${REPS:-2} TAG=${TAG}_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
fi
