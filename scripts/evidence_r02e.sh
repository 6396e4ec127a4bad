# round-2 final evidence: GPU tests, smoke, full bench (e2e + CPU arm), reference arm, launch list,
# ncu --set full of the attention backward per variant (roofline traffic), long-seq, configs[4] microbench
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r02e_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02e_bench_reference.json 2> gpurun_out/r02e_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_v4.csv python bench.py --blocks 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for v in msa_row msa_col pair_row pair_col; do
  case $v in msa_row) n=5;; msa_col) n=2;; *) n=3;; esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd|attn_dbias|attn_bias_transpose" -c $n -f -o gpurun_out/r02e_bwd_$v python scripts/attn_micro.py --variant $v --iters 1 > /dev/null 2>&1
done
for n in 1024 2048 4096; do timeout 900 python bench.py --workload longseq --n-res $n --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02e_longseq.jsonl
timeout 600 python scripts/kernel_microbench.py > gpurun_out/r02e_kernel_microbench.jsonl 2> gpurun_out/r02e_kernel_microbench.err
ls gpurun_out/
