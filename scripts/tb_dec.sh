for G in 89 148; do
./scripts/tma_bench_mla 2 $G 8 1; ./scripts/tma_bench_mla 4 $G 6 1; ./scripts/tma_bench_mla 4 $G 3 1; ./scripts/tma_bench_mla 8 $G 3 1
done
