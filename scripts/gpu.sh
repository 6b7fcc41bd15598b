#!/bin/bash
# One parametrised GPU-box runner (replaces the round-1 one-off scripts).
#   scripts/gpu.sh TAG STEP [STEP ...]
# STEP is one of
#   smoke                 __graft_entry__.smoke()
#   test:EXPR[:ARGS]      pytest -m EXPR ARGS (ARGS eval'd: quote -k expressions with '')
#   bench:CONFIG[:ARGS]   bench.py --config CONFIG (CONFIG "ref" = --impl reference)
#   launches:CONFIG       ncu launch list (gpu__time_duration) of one bench run
#   full:CONFIG:KERNEL[:COUNT[:ARGS]]  ncu --set full of KERNEL (regex) in a bench run
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
      cfg=${rest%%:*}; r2=${rest#*:}; kern=${r2%%:*}; cnt=1; fargs=""
      if [[ $r2 == *:* ]]; then r3=${r2#*:}; cnt=${r3%%:*}; [[ $r3 == *:* ]] && fargs=${r3#*:}; fi
      timeout 2400 ncu --set full --clock-control none --import-source on -k "regex:$kern" -c "$cnt" \
        -o "$OUT/$i.full_${cfg}" python bench.py --config "$cfg" --steps 1 --warmup 1 $fargs \
        > "$OUT/$i.full_$cfg.log" 2>&1 ;;
    py)
      scr=${rest%%:*}; args=""; [[ $rest == *:* ]] && args=${rest#*:}
      timeout 3000 python $scr $args > "$OUT/$i.py.log" 2>&1 ;;
    *) echo "unknown step $step"; continue ;;
  esac
  echo "step $i [$step] rc=$?"
done
for f in "$OUT"/*.log; do echo "== $f"; tail -4 "$f" | cut -c1-400; done
