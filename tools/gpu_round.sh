#!/bin/bash
# One GPU verification pass (run under gpurun from the repo root):
#   GPU parity tests, the bench line, the ncu launch list of one bench step,
#   and ncu --set full captures of the top kernels. Outputs -> gpurun_out/.
# Usage: tools/gpu_round.sh [tests] [bench] [launches] [full]   (default: all)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
what="${*:-tests bench launches full}"
nvidia-smi -L > gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt; lscpu | grep 'Model name' >> gpurun_out/gpu.txt
for w in $what; do case $w in
tests)
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  tail -5 gpurun_out/pytest_gpu.log ;;
smoke)
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
  tail -3 gpurun_out/smoke.log ;;
bench)
  timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
  cat gpurun_out/bench.json ;;
mb)
  ./tools/mb/f32x2.bin > gpurun_out/mb_f32x2.txt 2>&1; cat gpurun_out/mb_f32x2.txt ;;
ab)  # A/B of an engine option: CQG_OPTS for the second run, e.g. AB=exact_x2=0
  timeout 900 python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_a.json 2>&1
  CQG_OPTS="$AB" timeout 900 python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_b.json 2>&1
  python -c "
import json
for f in ['a','b']:
    d=json.loads(open(f'gpurun_out/bench_{f}.json').read().strip().splitlines()[-1])
    print(f, round(d['value']), {k: round(v['ms']) for k, v in sorted(d['roofline']['per_kernel'].items(), key=lambda kv: -kv[1]['ms'])[:8]})
" ;;
reference)
  timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
  cat gpurun_out/bench_ref.json ;;
launches)
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --ncu > gpurun_out/ncu_launches.log 2>&1
  echo "ncu launches exit $?"
  python tools/ncu_launch_summary.py gpurun_out/launches.csv gpurun_out/launches_summary.json | tail -30
  gzip -f gpurun_out/launches.csv ;;
full)
  for k in gemm_exact_big:20 gemm_fixup:400 gemm_tc_kernel:400 ln_warp:400 fold_kernel:400 kl_kernel:5 attention_warp:100; do
    pat=${k%%:*}; skip=${k##*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$pat -s $skip -c 2 \
      -o gpurun_out/prof_$pat -f python bench.py --ncu > gpurun_out/ncu_full_$pat.log 2>&1
    echo "ncu full $pat exit $?"
  done ;;
esac; done
