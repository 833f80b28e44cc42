cd /root/repo
export DQ_WAIT_TIMEOUT_S=15
for pdl in 0 1; do
DQ_PDL=$pdl timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2979$pdl tools/early_repro.py > gpurun_out/r2_early_repro_pdl$pdl.log 2>&1; echo R$pdl=$?; grep -E "ok=|rror" gpurun_out/r2_early_repro_pdl$pdl.log | head -8
done
