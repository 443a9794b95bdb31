for L in 0 1; do for G in 148 74; do
./scripts/tma_bench_mla 9 $G 3 $L; ./scripts/tma_bench_mla 3 $G 8 $L; ./scripts/tma_bench_mla 5 $G 5 $L; ./scripts/tma_bench_mla 1 $G 8 $L; ./scripts/tma_bench_mla 2 $G 8 $L
done; done
