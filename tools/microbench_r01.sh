# Microbenchmarks behind DESIGN.md section 6b (run on a B200 box; each prints one table).
set -e
cd "$(dirname "$0")"
for b in tmem_bw umma_rate commit_lat mbar_cost copy_lat pipe_bench; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_$b $b.cu
  echo "=== $b"; timeout 120 /tmp/mb_$b
done
