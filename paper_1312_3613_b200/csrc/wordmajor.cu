// csrc/wordmajor.cu -- device sort / run-length encoding for the word-major z-step order
// (lda.cu build_word_major): the local tokens sorted by (document block, word), and
// the (block, word) runs that become the z-step's work units. Built once per corpus.
#include <cstdint>

#include <cub/cub.cuh>

#include "common.cuh"

namespace bnmc_gpu {

// Stable sort of (key, value) pairs on key bits [0, end_bit). The buffers are a
// double buffer; returns which of them holds the sorted data (0: keys/vals, 1: alt).
int sort_pairs_u32(std::uint32_t* keys, std::uint32_t* keys_alt, int* vals, int* vals_alt, std::int64_t n,
                   int end_bit, cudaStream_t st) {
  cub::DoubleBuffer<std::uint32_t> k(keys, keys_alt);
  cub::DoubleBuffer<int> v(vals, vals_alt);
  std::size_t bytes = 0;
  BNMC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, static_cast<int>(n), 0, end_bit, st));
  DevBuf<unsigned char> tmp;
  tmp.alloc(bytes);
  BNMC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k, v, static_cast<int>(n), 0, end_bit, st));
  BNMC_CUDA(cudaStreamSynchronize(st));
  return k.Current() == keys ? 0 : 1;
}

// Runs of equal keys in a sorted array: unique keys and run lengths; returns the count.
std::int64_t run_length_u32(const std::uint32_t* keys, std::int64_t n, std::uint32_t* uniq, int* counts,
                            cudaStream_t st) {
  DevBuf<int> nruns;
  nruns.alloc(1);
  std::size_t bytes = 0;
  BNMC_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, keys, uniq, counts, nruns.p, static_cast<int>(n), st));
  DevBuf<unsigned char> tmp;
  tmp.alloc(bytes);
  BNMC_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, bytes, keys, uniq, counts, nruns.p, static_cast<int>(n), st));
  int h = 0;
  BNMC_CUDA(cudaMemcpyAsync(&h, nruns.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  BNMC_CUDA(cudaStreamSynchronize(st));
  return h;
}

}  // namespace bnmc_gpu
