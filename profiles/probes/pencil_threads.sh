for t in 1 2 4; do echo "KH_PENCIL_THREADS=$t"; KH_PENCIL_THREADS=$t python profiles/probes/e2e_full.py 2>&1 | grep "^total" | tail -2; done
