#!/bin/bash
# tools/gpu.sh — the one driver for GPU-side measurement runs (executed on the
# B200 box under gpurun, from the repo root; outputs land in gpurun_out/).
#
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu.sh TAG STEP [STEP ...]'
#
# Steps (run in the order given, each under its own timeout):
#   tests       pytest -m gpu (+ smoke)                 -> pytest_TAG.log, smoke_TAG.log
#   bench       bench.py defaults (coded + raw pass)    -> bench_TAG.log
#   quick       bench.py --steps 5 --warmup 3, no decode/cpu/raw -> bench_quick_TAG.log
#   ref         bench.py --impl reference               -> bench_ref_TAG.log
#   gauss       bench.py --init gaussian (quick)        -> bench_gauss_TAG.log
#   cpuattn     CPU attention placement, m = 1, 2, 4    -> bench_cpuattn_TAG.jsonl
#   configs     every BASELINE model shape (quick)      -> configs_TAG.jsonl
#   launches    ncu launch list of one timed step       -> launches_TAG.csv
#   full:REGEX  ncu --set full of one launch matching REGEX inside the timed step -> full_TAG_REGEX.ncu-rep
#   kbench:ARGS tools/kbench.py ARGS                    -> kbench_TAG.jsonl
#   sanitize    compute-sanitizer tier (pytest -m sanitizer) -> sanitize_TAG.log
set -u
TAG=${1:?tag}
shift
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
QUICK="--steps 5 --warmup 3 --no-cpu-baseline --no-decode --no-raw"
line() { grep '"metric"' "$1" | tail -1 | cut -c1-220; }
for step in "$@"; do
  case "$step" in
    tests)
      timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1
      echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
      echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log ;;
    bench)
      timeout 1500 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"; line gpurun_out/bench_$TAG.log ;;
    quick)
      timeout 900 python bench.py $QUICK > gpurun_out/bench_quick_$TAG.log 2>&1; echo "quick rc=$?"
      line gpurun_out/bench_quick_$TAG.log ;;
    ref)
      timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
      line gpurun_out/bench_ref_$TAG.log ;;
    gauss)
      timeout 900 python bench.py --init gaussian --steps 5 --warmup 3 --no-cpu-baseline --no-decode \
        > gpurun_out/bench_gauss_$TAG.log 2>&1; echo "gauss rc=$?"; line gpurun_out/bench_gauss_$TAG.log ;;
    cpuattn)
      : > gpurun_out/bench_cpuattn_$TAG.jsonl
      for m in 1 2 4; do
        timeout 900 python bench.py --attn-cpu --micro-batches $m $QUICK 2>/dev/null | grep '"metric"' \
          >> gpurun_out/bench_cpuattn_$TAG.jsonl; echo "cpuattn m=$m rc=$?"
      done ;;
    configs)
      : > gpurun_out/configs_$TAG.jsonl
      for cfg in "--model mixtral-8x7b" "--model mixtral-8x7b --cache-gb 5.25" "--model mixtral-8x7b --k 4" \
                 "--model dsv2-lite --cache-gb 5.25" "--model qwen2-57b --cache-gb 5.25" "--model mixtral-8x22b" \
                 "--model mixtral-8x7b --batch 1 --k 4 --moe-batching one" \
                 "--model dsv2-lite --batch 1 --k 4 --moe-batching one"; do
        timeout 1200 python bench.py $cfg $QUICK 2>/dev/null | grep '"metric"' >> gpurun_out/configs_$TAG.jsonl
        echo "config [$cfg] rc=$?"
      done ;;
    launches)
      SMO_PROFILE_TIMED=1 timeout 1200 $NCU --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode --no-raw > /dev/null 2>&1
      echo "ncu launches rc=$?" ;;
    full:*)
      rx=${step#full:}
      SMO_PROFILE_TIMED=1 timeout 1500 $NCU --profile-from-start off --set full --clock-control none \
        --import-source on -k regex:$rx -c 1 -o gpurun_out/full_${TAG}_$rx -f \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-decode --no-raw \
        > gpurun_out/ncu_full_${TAG}_$rx.log 2>&1
      echo "ncu full $rx rc=$?" ;;
    kbench:*)
      timeout 1500 python tools/kbench.py ${step#kbench:} > gpurun_out/kbench_$TAG.jsonl 2> gpurun_out/kbench_$TAG.err
      echo "kbench rc=$?"; tail -2 gpurun_out/kbench_$TAG.jsonl ;;
    sanitize)
      timeout 1800 python -m pytest tests -m sanitizer -q > gpurun_out/sanitize_$TAG.log 2>&1
      echo "sanitize rc=$?"; tail -3 gpurun_out/sanitize_$TAG.log ;;
    *) echo "unknown step $step" ;;
  esac
done
