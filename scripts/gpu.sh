#!/bin/bash
# One parametrised GPU-box runner (replaces the round-1 one-off scripts).
#   scripts/gpu.sh TAG STEP [STEP ...]
# STEP is one of
#   smoke                 __graft_entry__.smoke()
#   test:EXPR[:ARGS]      pytest -m EXPR ARGS (ARGS eval'd: quote -k expressions with '')
#   bench:CONFIG[:ARGS]   bench.py --config CONFIG (CONFIG "ref" = --impl reference)
#   launches:CONFIG       ncu launch list (gpu__time_duration) of one bench run
#   full:CONFIG:KERNEL[:COUNT[:SKIP[:ARGS]]]  ncu --set full of KERNEL (regex) in a bench run
#                         (COUNT launches after skipping SKIP matching ones)
#   lite:...              as full:, without the instrumented source-counter passes
#   shard1[:ENV=V ...]    bench.py under torchrun with one rank (world-1 sharded C3 over NCCL)
#   py:SCRIPT[:ARGS]      python SCRIPT ARGS
# Logs go to gpurun_out/TAG/; the parity log to gpurun_out/TAG/parity.jsonl.
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export RPLU_PARITY_LOG=$OUT/parity.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > "$OUT/gpu.txt"
i=0
for step in "$@"; do
  i=$((i + 1))
  kind=${step%%:*}; rest=${step#*:}
  case $kind in
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/$i.smoke.log" 2>&1 ;;
    test)
      expr=${rest%%:*}; args=""; [[ $rest == *:* ]] && args=${rest#*:}
      eval "timeout 3000 python -m pytest -m \"$expr\" -q -rs $args" > "$OUT/$i.test.log" 2>&1 ;;
    bench)
      cfg=${rest%%:*}; args=""; [[ $rest == *:* ]] && args=${rest#*:}
      if [[ $cfg == ref ]]; then
        timeout 1200 python bench.py --impl reference $args > "$OUT/$i.bench_ref.log" 2>&1
      else
        timeout 1200 python bench.py --config "$cfg" $args > "$OUT/$i.bench_$cfg.log" 2>&1
      fi ;;
    launches)
      timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
        --log-file "$OUT/$i.launches_$rest.csv" python bench.py --config "$rest" --steps 1 --warmup 3 \
        > "$OUT/$i.launches_$rest.log" 2>&1 ;;
    full)
      cfg=${rest%%:*}; r2=${rest#*:}; kern=${r2%%:*}; cnt=1; skip=0; fargs=""
      if [[ $r2 == *:* ]]; then r3=${r2#*:}; cnt=${r3%%:*};
        if [[ $r3 == *:* ]]; then r4=${r3#*:}; skip=${r4%%:*}; [[ $r4 == *:* ]] && fargs=${r4#*:}; fi; fi
      timeout 2400 ncu --set full --clock-control none --import-source on -k "regex:$kern" -s "$skip" -c "$cnt" \
        -o "$OUT/$i.full_${cfg}" python bench.py --config "$cfg" --steps 1 --warmup 1 $fargs \
        > "$OUT/$i.full_$cfg.log" 2>&1 ;;
    lite)   # as full, without the instrumented (SourceCounters) passes: for multi-second kernels
      cfg=${rest%%:*}; r2=${rest#*:}; kern=${r2%%:*}; cnt=1; skip=0; fargs=""
      if [[ $r2 == *:* ]]; then r3=${r2#*:}; cnt=${r3%%:*};
        if [[ $r3 == *:* ]]; then r4=${r3#*:}; skip=${r4%%:*}; [[ $r4 == *:* ]] && fargs=${r4#*:}; fi; fi
      timeout 2400 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis \
        --section MemoryWorkloadAnalysis --section InstructionStats --section LaunchStats \
        --section Occupancy --section SchedulerStats --section WarpStateStats \
        --clock-control none -k "regex:$kern" -s "$skip" -c "$cnt" \
        -o "$OUT/$i.lite_${cfg}" python bench.py --config "$cfg" --steps 1 --warmup 1 $fargs \
        > "$OUT/$i.lite_$cfg.log" 2>&1 ;;
    shard1)   # world-1 sharded C3 over NCCL (torchrun, one rank); rest = env assignments
      envs=""; [[ $rest != shard1 ]] && envs=$rest
      env RPLU_FORCE_SHARDED=1 $envs timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
        --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 2 --warmup 1 \
        > "$OUT/$i.shard1.log" 2>&1 ;;
    py)
      scr=${rest%%:*}; args=""; [[ $rest == *:* ]] && args=${rest#*:}
      timeout 3000 python $scr $args > "$OUT/$i.py.log" 2>&1 ;;
    *) echo "unknown step $step"; continue ;;
  esac
  echo "step $i [$step] rc=$?"
done
for f in "$OUT"/*.log; do echo "== $f"; tail -4 "$f" | cut -c1-400; done
