# GEMM tiling A/B on the merge shapes: HPS_GEMM64=0 (128x128 one CTA/SM) vs 1 (64x64 paired fragments)
for v in 1; do echo "== HPS_GEMM64=$v"; HPS_GEMM64=$v python -c "
import sys; sys.path.insert(0, '.')
from tools.bench_inverse import t_gemm
for s in [(4096,4096,1024,1),(1024,4096,1024,1),(3072,3072,512,2),(512,3072,512,2),(1536,1536,256,8),(256,1536,256,8),(128,768,128,32),(16384,16384,4096,1),(4096,16384,4096,1)]: t_gemm(*s)
" 2>&1; done
