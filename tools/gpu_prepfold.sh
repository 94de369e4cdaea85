# prep folded into conv1's idle warp: full GPU tests, then cfg1 / cfg3 kernel lists and bench, fold on / off
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/pf
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pf/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pf/pytest.log
for v in 1 0 1 0; do
  BP_PREP_FOLD=$v timeout 300 python tools/graph_kernels.py 5 cfg1 > gpurun_out/pf/gk_cfg1_$v.txt 2>&1
  echo "fold=$v"; grep -E "^  [0-2] |step span" gpurun_out/pf/gk_cfg1_$v.txt | cut -c1-110
done
for v in 1 0; do
  BP_PREP_FOLD=$v BP_BENCH_NO_CFG4=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pf/bench_$v.log 2>&1
  tail -1 gpurun_out/pf/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fold', $v, d['ms_per_step'], d['e2e']['ms_per_step'], d['lstm'].get('ms_per_step'))"
done
