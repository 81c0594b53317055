# One GPU evidence pass: parity tests, smoke, bench (both arms), configs 3-5,
# per-CTA timelines, ncu launch list + full captures of the GEMVs and the
# latency-bound kernels.  TAG names the round (outputs in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
timeout 1500 python scripts/configs_report.py $TAG > gpurun_out/configs_$TAG.log 2>&1
for cfg in mixtral olmoe qwen15; do
  timeout 600 python scripts/cta_timeline.py $cfg 0,4,8 $TAG > gpurun_out/tl_${cfg}_$TAG.txt 2>&1
done
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/profile_step.py --ks 0,8 > gpurun_out/prof_launch_$TAG.log 2>&1
echo "ncu1 rc=$?" >> gpurun_out/prof_launch_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"stream_gemv|dense_gemv_cluster|expert_ffn" -c 10 -o gpurun_out/gemv_full_$TAG python scripts/profile_step.py --ks 8 --layers 2 > gpurun_out/prof_full_$TAG.log 2>&1
echo "ncu2 rc=$?" >> gpurun_out/prof_full_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"moe_route|moe_combine|attn_partial|attn_combine" -c 8 -o gpurun_out/small_full_$TAG python scripts/profile_step.py --ks 0 --layers 2 > gpurun_out/prof_small_$TAG.log 2>&1
echo "ncu3 rc=$?" >> gpurun_out/prof_small_$TAG.log
fi
