# prep fold A/B: kernel lists (cfg1, cfg3, inf1), fold on / off, alternating
mkdir -p gpurun_out/pf
for v in 1 0 1 0; do
  for w in cfg1 cfg3 inf1; do BP_PREP_FOLD=$v timeout 300 python tools/graph_kernels.py 10 $w > gpurun_out/pf/gk_${w}_$v.txt 2>&1; done
  echo "fold=$v"; for w in cfg1 cfg3 inf1; do grep -E "step span" gpurun_out/pf/gk_${w}_$v.txt; done
  grep -E "^  [0-1] " gpurun_out/pf/gk_cfg1_$v.txt | cut -c1-100
done
