# A/B of the attention row-block threshold (alternating, 2 rounds)
for round in 1 2; do
for lib in "$@"; do
  for args in "--w 4 --ctx 1500" "--w 4 --ctx 3000" "--w 4 --ctx 6000" "--w 8 --ctx 3000" "--w 2 --ctx 3000"; do
    PS_LIB=$lib python scripts/pass_time.py --shape llama3.1-8b $args --reps 10 2>&1 | tail -1 | sed "s|^|$(basename $lib) |"
  done
done
done
