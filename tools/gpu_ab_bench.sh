# same-box A/B of one source file on the bench (device step + e2e): B = working tree, A = ab_old/<file>
F=$1
mkdir -p gpurun_out/abb
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/abb/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/abb/pytest.log
run() { BP_BENCH_NO_CFG4=1 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abb/$V.log 2>&1; tail -1 gpurun_out/abb/$V.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V', round(d['ms_per_step'],4), round(d['e2e']['ms_per_step'],4), round(d['lstm'].get('ms_per_step',0),4))"; }
V=B; run; run
cp paper_1910_03552_b200/libbeast_b200.so /tmp/libB.so; cp paper_1910_03552_b200/csrc/$F /tmp/srcB
cp ab_old/$F paper_1910_03552_b200/csrc/$F
python -m paper_1910_03552_b200.build > gpurun_out/build2.log 2>&1 || exit 1
V=A; run; run
cp /tmp/libB.so paper_1910_03552_b200/libbeast_b200.so; cp /tmp/srcB paper_1910_03552_b200/csrc/$F
V=B; run
