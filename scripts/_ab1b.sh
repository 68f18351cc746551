# A/B of library builds on the 1B draft step (and the 8B verify pass), alternating, 2 rounds
for round in 1 2; do
for lib in "$@"; do
  PS_LIB=$lib python scripts/pass_time.py --shape llama3.2-1b --w 0 2>&1 | tail -1 | sed "s|^|$lib |"
  PS_LIB=$lib python scripts/pass_time.py --shape llama3.1-8b --w 4 2>&1 | tail -1 | sed "s|^|$lib |"
done
done
