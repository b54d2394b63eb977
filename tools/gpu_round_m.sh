mkdir -p gpurun_out
cd tools
timeout 120 python pf_timing.py > ../gpurun_out/m_pft.log 2>&1
timeout 120 python pf_timing.py 4096 14336 16 2048 base >> ../gpurun_out/m_pft.log 2>&1
timeout 120 python pf_timing.py 14336 4096 16 2048 >> ../gpurun_out/m_pft.log 2>&1
