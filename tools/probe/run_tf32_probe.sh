cd $GRAFT_REPO_ROOT
timeout 60 ./tools/probe/tf32_probe_trace 16384 16384 512 1 2 64 | tail -12
for args in "1000 777 64 3" "2048 2048 256 3" "4096 4096 512 3" "16384 16384 512 3 5 16" "16384 16384 512 1 5 16" "65536 65536 512 3 3 128" "65536 65536 512 1 3 128" "8192 65536 512 3 5 64"; do
  echo "== $args"; timeout 120 ./tools/probe/tf32_probe $args | grep "avg\|max"; echo "rc=$?"
done
