set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r01_launches_v7.csv python bench.py --blocks 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev_bench.log 2>&1
for v in msa_row msa_col pair_row pair_col; do
  case $v in msa_row) n=5;; msa_col) n=2;; *) n=3;; esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd|attn_dbias|attn_bias_transpose" -c $n -f -o gpurun_out/r01_bwd_v3_$v python scripts/attn_micro.py --variant $v --iters 1 > /dev/null 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_fwd" -c 1 -f -o gpurun_out/r01_fwd_v3_$v python scripts/attn_micro.py --variant $v --iters 1 --bwd 0 > /dev/null 2>&1
done
python scripts/kernel_microbench.py --out gpurun_out/r01_kernel_microbench_v5.jsonl > /dev/null 2>&1
ls -la gpurun_out/
