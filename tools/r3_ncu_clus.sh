cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/n
for c in cfg1 cfg2; do
python tools/scan_ab.py --config $c --steps 3 --head cluster > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:clus_topk -s 6 -c 1 -o gpurun_out/n/clus_$c python tools/scan_ab.py --config $c --steps 3 --head cluster > gpurun_out/n/ncu_$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:attend_cand -s 6 -c 1 -o gpurun_out/n/att_cfg2 python tools/scan_ab.py --config cfg2 --steps 3 --head kth > gpurun_out/n/ncu_att.log 2>&1
ls -la gpurun_out/n
