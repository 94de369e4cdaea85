python -m paper_1910_03552_b200.build > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for args in "1 0 x0 2592" "1 0 nox0 2592" "1 0 x0 41472" "1 0 nox0 41472" "1 1 x0 41472" "1 2 x0 41472" "1 3 x0 41472"; do
  echo "### $args"; timeout 120 python tools/conv1_trace.py $args 2>&1 | tail -9
done
