cd $GRAFT_REPO_ROOT
for ck in 0 256 128 64; do for args in "4096 65536 256 3 0 16 0 1" "4096 65536 256 3 0 16 0 0"; do
  echo "== chunk $ck $args"; CHUNK_KB=$ck timeout 120 ./tools/probe/tf32_probe $args | grep "max"
done; done
for args in "65536 65536 512 3 3 128" "65536 65536 512 1 3 128" "16384 16384 512 3 5 16" "1000 777 64 3" "4096 4096 512 3"; do
  echo "== $args"; timeout 120 ./tools/probe/tf32_probe $args | grep "max\|avg"
done
