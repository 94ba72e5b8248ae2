for it in 4 6 8 10 14; do
  echo "LP iters $it"; IGP_LP_ITERS=$it timeout 600 python tools/config_times.py headline_community,large_community 2>&1 | grep -v "^$"
done
