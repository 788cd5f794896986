# rows-DMMA kernel variants (development aid; build/variants/*.so built by paper_1609_00076_b200.build --out=)
P=tools/rows_dmma_probe.py
S="4x8192x8192 8x8192x8192 16x8192x8192 32x8192x8192 16x4096x4096 8x32768x8192 16x65536x2048"
timeout 300 python $P > gpurun_out/rd_main.log 2>&1
for ct in 1 2 4; do MY_DGEMM_RD_CT=$ct timeout 200 python $P $S > gpurun_out/rd_ct$ct.log 2>&1; done
for v in build/variants/*.so; do b=$(basename $v .so); for ct in 2 4; do MY_DGEMM_RD_CT=$ct MY_DGEMM_LIB=$PWD/$v timeout 200 python $P $S > gpurun_out/${b}_ct$ct.log 2>&1; done; done
