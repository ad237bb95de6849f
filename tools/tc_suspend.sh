# mbarrier try_wait suspend-time hint: K1-TC (cfg4 t=16) and K1-TC-sym (cfg4 t=1)
for ns in 0 2000 20000 200000; do
  echo "NS=$ns $(LGP_TC_SUSPEND_NS=$ns timeout 100 python tools/profile_k1.py --t 16 --reps 3 2>&1 | tail -1)"
  echo "NS=$ns $(LGP_TC_SUSPEND_NS=$ns timeout 100 python tools/profile_k1.py --t 1 --reps 3 2>&1 | tail -1)"
done
