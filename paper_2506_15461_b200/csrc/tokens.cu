// Synthetic, learnable token stream for the LLaMA block (SURVEY §7 hard part 6):
// addressed purely by (data_seed, stream, index) like the reference's batches
// (src/dataset.cpp:15-20), integer-only -> bit-exact between the CPU oracle
// (oracle/llama_oracle.py::token_batch) and the GPU.
//
// Row r of a batch is T+1 tokens.  Draw j of row r uses counter c = r*(T+1)+j+1
// of key = derive_key(data_seed, stream, index):  bits = mix64(key + c*phi).
//   j == 0, or bits>>62 == 3 (1 in 4):  skewed unigram  ((lo32 % V) * (hi32 % V)) / V
//   otherwise:                          sparse bigram   succ(prev, (bits >> 40) & 3)
// with succ(v, c) = mix64(derive_key(data_seed, 4) ^ (4v + c)) % V.
#include "common.cuh"

namespace ckf {

__host__ __device__ __forceinline__ uint32_t token_draw(uint64_t key, uint64_t succ_key, uint64_t counter,
                                                       uint32_t prev, bool first, uint64_t V) {
  const uint64_t bits = mix64(key + counter * 0x9e3779b97f4a7c15ULL);
  if (first || (bits >> 62) == 3) {
    const uint64_t a = (bits & 0xffffffffULL) % V, b = (bits >> 32) % V;
    return static_cast<uint32_t>((a * b) / V);
  }
  const uint64_t c = (bits >> 40) & 3ULL;
  return static_cast<uint32_t>(mix64(succ_key ^ (4ULL * prev + c)) % V);
}

namespace {
__global__ void token_kernel(uint64_t key, uint64_t succ_key, size_t rows, size_t T, uint64_t V, int* __restrict__ out) {
  const size_t r = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  uint32_t prev = 0;
  int* row = out + r * (T + 1);
  for (size_t j = 0; j <= T; ++j) {
    prev = token_draw(key, succ_key, r * (T + 1) + j + 1, prev, j == 0, V);
    row[j] = static_cast<int>(prev);
  }
}
}  // namespace

void llama_token_batch(uint64_t data_seed, uint64_t stream, uint64_t index, size_t rows, size_t T, size_t V,
                       int* out, cudaStream_t s) {
  const uint64_t key = derive_key(data_seed, stream, index);
  const uint64_t succ_key = derive_key(data_seed, 4);
  token_kernel<<<grid_for(rows, 64, 1 << 20), 64, 0, s>>>(key, succ_key, rows, T, V, out);
  CKF_LAUNCH_CHECK();
}

}  // namespace ckf
