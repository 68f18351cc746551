for lib in scratch/lib_base.so scratch/lib_pre.so scratch/lib_pre_ml_q.so scratch/lib_step.so; do
  for i in 1 2 3; do
    echo "$lib run $i: $(PS_LIB=$lib timeout 300 python -m pytest tests/test_gpu_pipeline.py -x -q 2>&1 | tail -1)"
  done
done
PS_LIB=scratch/lib_step.so timeout 300 python -m pytest tests/test_gpu_pipeline.py -x -q 2>&1 | grep -E "Error|assert" | head -20
