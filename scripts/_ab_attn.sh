# A/B of library builds on the attention-heavy points (alternating, 2 rounds)
for round in 1 2; do
for lib in "$@"; do
  for args in "--shape llama3.1-8b --w 4 --ctx 600" "--shape llama3.2-1b --w 0 --ctx 600" "--shape llama3.1-8b --w 4 --ctx 8192" "--shape llama3.1-8b --w 0 --ctx 8192" "--shape llama3.1-8b --w 4 --ctx 32000" "--shape llama3.1-8b --w 16 --ctx 8192"; do
    PS_LIB=$lib python scripts/pass_time.py $args --reps 10 2>&1 | tail -1 | sed "s|^|$(basename $lib) |"
  done
done
done
