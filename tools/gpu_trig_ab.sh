# A/B: early PDL triggers in vt3 / pack_g (B = with, A = without), same box, alternating runs
mkdir -p gpurun_out/tr
python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do for w in cfg1 cfg3; do timeout 300 python tools/graph_kernels.py 10 $w > gpurun_out/tr/B_${w}_$i.txt 2>&1; echo "B $w $(grep 'step span' gpurun_out/tr/B_${w}_$i.txt)"; done; done
cp paper_1910_03552_b200/libbeast_b200.so /tmp/libB.so
python - <<'PY'
for p, old in (("paper_1910_03552_b200/csrc/network.cu", "  pdl_trigger();  // the heads data-gradient GEMM may set up (it waits for this kernel)\n"),
               ("paper_1910_03552_b200/csrc/vtrace_tile.cu", "  pdl_trigger();\n  pdl_wait();")):
    s = open(p).read(); assert old in s
    s = s.replace(old, "" if "heads" in old else "  pdl_wait();", 1); open(p, "w").write(s)
PY
python -m paper_1910_03552_b200.build > gpurun_out/build2.log 2>&1 || exit 1
for i in 1 2; do for w in cfg1 cfg3; do timeout 300 python tools/graph_kernels.py 10 $w > gpurun_out/tr/A_${w}_$i.txt 2>&1; echo "A $w $(grep 'step span' gpurun_out/tr/A_${w}_$i.txt)"; done; done
cp /tmp/libB.so paper_1910_03552_b200/libbeast_b200.so
for w in cfg1 cfg3; do timeout 300 python tools/graph_kernels.py 10 $w > gpurun_out/tr/B_${w}_3.txt 2>&1; echo "B $w $(grep 'step span' gpurun_out/tr/B_${w}_3.txt)"; done
