cd $GRAFT_REPO_ROOT
for cfg in "PF_TF32_PFDIST=0 PF_TF32_CHUNK_KB=128" "PF_TF32_PFDIST=0 PF_TF32_CHUNK_KB=256"; do
  for np in 1 3; do echo "== $cfg npass $np"; env $cfg timeout 100 ./tools/probe/tf32_probe 65536 65536 512 $np 3 128 | grep -E "avg|max"; done
done
