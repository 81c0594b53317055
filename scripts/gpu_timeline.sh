# Per-CTA timelines under env variants: TL_VARIANTS="name:ENV=V,ENV2=V;name2:..." TL_CFGS="mixtral olmoe"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in ${TL_CFGS:-mixtral}; do
  IFS=';' read -ra VS <<< "${TL_VARIANTS:-base:X=1}"
  for v in "${VS[@]}"; do
    name=${v%%:*}; envs=${v#*:}
    env ${envs//,/ } timeout 600 python scripts/cta_timeline.py $cfg ${TL_KS:-0,8} $name > gpurun_out/tl_${cfg}_$name.txt 2>&1
  done
done
