cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py tests/test_gpu_rope_fused.py -q -x -k "decode and not mla" -p no:cacheprovider > gpurun_out/pair16_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/pair16_tests.log)"
for rep in 1 2; do
echo "== pair16"; timeout 300 python scripts/microbench.py --kernel decode --bs 16 --budgets 44,89,104,148 --layers 8 2>&1 | tail -4
echo "== single"; SEMIPD_DECODE_SINGLE=1 timeout 300 python scripts/microbench.py --kernel decode --bs 16 --budgets 44,89,104,148 --layers 8 2>&1 | tail -4
done
