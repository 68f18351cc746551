# attention n-tiles per row block forced to 1 / 2 / 3 (any choice gives identical rows): pass times
for lib in "$@"; do
  for ctx in 1024 2048 4096 8192 16384; do
    for w in 2 4 8 16; do
      PS_LIB=$lib python scripts/pass_time.py --shape llama3.1-8b --w $w --ctx $ctx --reps 6 2>&1 | tail -1 | sed "s|^|$(basename $lib) |"
    done
  done
done
