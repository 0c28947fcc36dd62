cd "${GRAFT_REPO_ROOT}"
for L in libp2s_k6.so libp2s_k7.so libp2s_k8.so libp2s_k9.so; do for S in 3 4; do
P2S_BLUR_STAGES=$S P2S_LIB_NAME=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(\"$L stages $S\", round(d[\"value\"],1), round(d[\"stages\"][\"k_blur\"][\"ms_per_launch\"],3), d['clocks']['sm_mhz'])"
done; done
