# k / time of large 4-D problems with the deterministic (Frobenius) stop vs the spectral screen
for cfg in "" "HB_SPECTRAL=1" "HB_SPECTRAL=1 HB_SCREEN_GATE=1e9"; do
  echo "== $cfg"
  for prob in "4 2 exp_neg_r 32000" "4 1 exp_neg_r 32000" "4 3 exp_neg_r 16000"; do
    env $cfg HB_DEBUG_STOP=1 timeout 300 python tools/profile_one.py $prob 1 2>&1 | tail -4
  done
done
