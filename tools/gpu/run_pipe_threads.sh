for th in 1 2 3 4 8; do echo "threads $th"; MSURF_PIPELINE_THREADS=$th python tools/gpu/e2e_profile3.py 2>&1 | grep "chunk 32" | tail -2; done
