bash exp/ncu_cap.sh medium ammmse_solve --per-block 256
bash exp/ncu_cap.sh massive ammmse_cluster --config massive --per-block 64
