for f in "" 1; do echo "cfg2 STKG_FUSED=$f"; STKG_FUSED=$f python tools/solve_time.py --cfg cfg2 --reps 20 | cut -c1-260; done
