cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KTC_LINEINFO=1
G2="gemm:2048:KWG=32;KWI=8;MDIMA=16;MDIMC=8;MWG=128;NDIMB=16;NDIMC=16;NWG=128;SA=1;SB=1;STRM=1;STRN=1;VWM=4;VWN=4"
G4="gemm:4096:KWG=16;KWI=8;MDIMA=16;MDIMC=8;MWG=128;NDIMB=16;NDIMC=8;NWG=64;SA=1;SB=1;STRM=1;STRN=1;VWM=2;VWN=4"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_k -c 1 -o gpurun_out/prof_g2048_r01b python tools/profile_winners.py "$G2" > gpurun_out/prof_g2048.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_k -c 1 -o gpurun_out/prof_g4096_r01b python tools/profile_winners.py "$G4" > gpurun_out/prof_g4096.log 2>&1
cat > /tmp/cb.py <<'PY'
import torch
torch.backends.cuda.matmul.allow_tf32 = False
for n in (2048, 4096):
    A = torch.rand(n, n, device="cuda"); B = torch.rand(n, n, device="cuda")
    C = A @ B
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:"gemm|sgemm|Kernel" -c 2 -o gpurun_out/prof_cublas_r01b python /tmp/cb.py > gpurun_out/prof_cublas.log 2>&1
ls -la gpurun_out/*.ncu-rep
tail -3 gpurun_out/prof_cublas.log
