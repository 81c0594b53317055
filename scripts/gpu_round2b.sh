# Round-2 (second session) GPU evidence pass (one gpurun call): parity tests, smoke, both bench
# arms with the driver's flags, configs 3-5, CTA timelines, ncu launch list,
# full captures (GEMVs, FFN traffic with provenance, small kernels).
# TAG names the pass (outputs in gpurun_out/$TAG/).
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02b}
O=gpurun_out/$TAG
mkdir -p $O
COMMIT=$(cat .commit 2>/dev/null || echo unknown)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=20 > $O/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
echo "smoke rc=$?" >> $O/smoke.txt
( time timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $O/bench_reference.json 2> $O/bench_reference.err
( time timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 ) > $O/bench_ours.json 2> $O/bench_ours.err
timeout 600 python bench.py > $O/bench_default_flags.json 2> $O/bench_default_flags.err
timeout 1800 python scripts/configs_report.py $TAG > $O/configs.log 2>&1
mv gpurun_out/configs_$TAG.json $O/configs.json 2>/dev/null
for cfg in mixtral olmoe qwen15; do
  timeout 600 python scripts/cta_timeline.py $cfg 0,4,8 $TAG > $O/cta_timeline_$cfg.txt 2>&1
done
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches.csv python scripts/profile_step.py --ks 0,8 > $O/prof_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:expert_ffn -c 1 -o $O/ffn_traffic python scripts/profile_step.py --ks 8 --layers 2 > $O/prof_ffn.log 2>&1
python scripts/ncu_traffic.py $O/ffn_traffic.ncu-rep $O/prof_ffn.log mixtral 8 "$COMMIT" \
  "ncu --set full --clock-control none -k regex:expert_ffn -c 1 python scripts/profile_step.py --ks 8 --layers 2" \
  $O/ncu_expert_traffic.json > $O/ncu_traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:expert_ffn_ring -c 1 -o $O/ffn_ring_traffic python scripts/profile_step.py --ks 4 --layers 2 > $O/prof_ffn_ring.log 2>&1
python scripts/ncu_traffic.py $O/ffn_ring_traffic.ncu-rep $O/prof_ffn_ring.log mixtral 4 "$COMMIT" \
  "ncu --set full --clock-control none -k regex:expert_ffn_ring -c 1 python scripts/profile_step.py --ks 4 --layers 2" \
  $O/ncu_expert_ring_traffic.json > $O/ncu_ring_traffic.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"dense_gemv_cluster|expert_ffn|stream_gemv" -c 10 -o $O/gemv_full python scripts/profile_step.py --ks 0,8 --layers 2 > $O/prof_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"moe_route|moe_combine|attn_partial|attn_combine" -c 8 -o $O/small_full python scripts/profile_step.py --ks 0 --layers 2 > $O/prof_small.log 2>&1
fi
# summarise the full captures here and keep the reports off the copy-back (64 MiB cap)
for r in gemv_full small_full ffn_traffic ffn_ring_traffic; do
  [ -f $O/$r.ncu-rep ] && python scripts/ncu_summary.py $O/$r.ncu-rep $O/ncu_$r.csv > /dev/null 2>&1
  [ -f $O/$r.ncu-rep ] && ncu -i $O/$r.ncu-rep --page details --csv > $O/ncu_${r}_details.csv 2>/dev/null
  mkdir -p /tmp/ncu_reps && mv $O/$r.ncu-rep /tmp/ncu_reps/ 2>/dev/null
done
du -sh $O > $O/size.txt
echo done > $O/DONE
