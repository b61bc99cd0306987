# A/B of the two-step producer's L2 prefetch distance (YB_TB2_PF) and stage count on configs 4, 3, 2
for rep in 1 2; do for pf in 0 1 2 4; do
  for g in "1024 1024 512 4" "512 512 512 2" "256 256 256 1"; do
    YB_TB2_PF=$pf timeout 300 python tools/stage_ab2.py $g 2>&1 | tail -4 | sed "s/^/pf=$pf /" | grep "stages=$(echo $g | awk '{print ($4==2)?2:3}')" | head -1
  done
done; done
