cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sl
python tools/shard_stage.py --shards 8 --steps 2 > gpurun_out/sl/plain.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv \
    -k regex:"sample|threshold|scan_tc|kth|attend|clus_topk|narrow|shard_merge|finalize|sort" \
    --log-file gpurun_out/sl/r3_shard_g8_launches.csv python tools/shard_stage.py --shards 8 --steps 2 > gpurun_out/sl/ncu.log 2>&1
