bash scripts/_ab.sh scratch/lib_s8.so scratch/lib_s6v.so scratch/lib_s5v.so
