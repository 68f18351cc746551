# attention keys per work item (sc x 64-key chunks, a per-stage constant) forced: pass times
for lib in "$@"; do
  for ctx in 4096 8192 16384 32000; do
    for w in 0 4 8; do
      PS_LIB=$lib python scripts/pass_time.py --shape llama3.1-8b --w $w --ctx $ctx --reps 6 2>&1 | tail -1 | sed "s|^|$(basename $lib) |"
    done
  done
done
