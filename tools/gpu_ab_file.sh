# same-box A/B of one source file: B = the working tree, A = ab_old/<file> (args: FILE WORKLOADS...)
F=$1; shift
mkdir -p gpurun_out/ab
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab/pytest.log
run() { for w in "$@"; do timeout 300 python tools/graph_kernels.py 10 $w > gpurun_out/ab/$V.$w.txt 2>&1; echo "$V $w $(grep 'step span' gpurun_out/ab/$V.$w.txt)"; done; }
V=B; run "$@"; run "$@"
cp paper_1910_03552_b200/libbeast_b200.so /tmp/libB.so; cp paper_1910_03552_b200/csrc/$F /tmp/srcB
cp ab_old/$F paper_1910_03552_b200/csrc/$F
python -m paper_1910_03552_b200.build > gpurun_out/build2.log 2>&1 || exit 1
V=A; run "$@"; run "$@"
cp /tmp/libB.so paper_1910_03552_b200/libbeast_b200.so; cp /tmp/srcB paper_1910_03552_b200/csrc/$F
V=B; run "$@"
