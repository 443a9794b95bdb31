cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 3000 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not cfg4 and not controller_loop and not multi_nccl and not nccl_graph and not peer_gather" > gpurun_out/r2_memcheck_all.log 2>&1; echo "memcheck all rc $?"
tail -3 gpurun_out/r2_memcheck_all.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_rope_fused.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "fused_rope_prefill_cfg2 or prefill_mla_latent" > gpurun_out/r2_racecheck.log 2>&1; echo "racecheck rc $?"
grep -E "passed|RACECHECK SUMMARY|ERROR SUMMARY" gpurun_out/r2_racecheck.log | tail -3
