# round-2 evidence, second pass (after the msa_row backward reordering and the TS-mode dK):
# launch list of bench.py --blocks 2, ncu --set full of one attention backward call per variant
# (roofline traffic), configs[4] microbench, long-seq 48-block forward.  Outputs under gpurun_out/.
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_v2.csv python bench.py --blocks 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for v in msa_row msa_col pair_row pair_col; do
  case $v in msa_row) n=5;; msa_col) n=2;; *) n=3;; esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd|attn_dbias|attn_bias_transpose" -c $n -f -o gpurun_out/r02b_bwd_$v python scripts/attn_micro.py --variant $v --iters 1 > /dev/null 2>&1
done
timeout 600 python scripts/kernel_microbench.py > gpurun_out/r02_kernel_microbench_v2.jsonl 2> gpurun_out/r02_kernel_microbench_v2.err
for n in 1024 2048 4096; do timeout 900 python bench.py --workload longseq --n-res $n --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02_longseq_v4.jsonl
ls gpurun_out/
