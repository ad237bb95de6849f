# per-CTA overhead probe: K1-TC time vs number of column segments (CTAs = 782 x segments)
for s in 7 14 28 56; do echo "SEG=$s $(LGP_TC_G=8 LGP_SEGMENTS=$s timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"; done
