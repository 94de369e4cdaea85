for args in "1 0 x0 41472" "1 0 nox0 41472" "1 1 x0 41472" "1 2 x0 41472"; do
  echo "### $args"; timeout 120 python tools/conv1_trace.py $args 2>&1 | grep -v Warn | tail -14
done
