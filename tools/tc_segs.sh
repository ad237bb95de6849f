# per-CTA overhead probe: K1-TC time vs number of column segments (CTAs = 782 x segments)
for s in 4 7 14 28; do echo "SEG=$s $(LGP_SEGMENTS=$s timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"; done
