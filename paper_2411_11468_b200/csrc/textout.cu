// write_membership (io.hpp:12, io.cpp:9-14) with the text formatted on the device:
// `vertex<TAB>label\n` for every vertex in id order. At R27 that is 134M lines (~2.3 GB
// of text); one thread per line computes its length, a scan places the lines, and a
// second pass writes the digits. Lines go through in batches of kBatch so the text
// buffer stays bounded, double-buffered so the D2H copy and fwrite of one batch
// overlap the formatting of the next. Same bytes as the reference's ofstream output.
#include <cub/cub.cuh>

#include <cstdio>
#include <string>

#include "internal.hpp"

namespace nulpa {
namespace {

constexpr uint64_t kBatch = uint64_t(1) << 24;  // lines per batch (<= 22 B of text each)

__device__ __forceinline__ uint32_t digits10(uint64_t v) {
  uint32_t d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

__device__ __forceinline__ void put10(char* end, uint64_t v) {
  do {
    *--end = char('0' + v % 10);
    v /= 10;
  } while (v);
}

__global__ void k_line_lengths(const uint32_t* __restrict__ labels, uint64_t first, uint64_t k,
                               uint32_t* __restrict__ len) {
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < k;
       t += uint64_t(gridDim.x) * blockDim.x)
    len[t] = digits10(first + t) + digits10(labels[t]) + 2;
}

__global__ void k_format_lines(const uint32_t* __restrict__ labels, uint64_t first, uint64_t k,
                               const uint64_t* __restrict__ at, char* __restrict__ out) {
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < k;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t v = first + t;
    char* p = out + at[t];
    const uint32_t dv = digits10(v);
    put10(p + dv, v);
    p[dv] = '\t';
    const uint32_t dl = digits10(labels[t]);
    put10(p + dv + 1 + dl, labels[t]);
    p[dv + 1 + dl] = '\n';
  }
}

struct Buffers {
  uint32_t* lab = nullptr;
  uint32_t* len = nullptr;
  uint64_t* at = nullptr;  // kBatch + 1 entries
  char* text = nullptr;
  char* host = nullptr;    // pinned
  void* scan_tmp = nullptr;
  size_t scan_bytes = 0;
};

}  // namespace

void write_membership_device(const char* path, const uint32_t* labels, uint64_t n, int device) {
  use_device(device);
  std::FILE* fp = std::fopen(path, "wb");
  if (!fp) throw Error(NULPA_EINVAL, std::string("cannot open output file: ") + path);
  cudaStream_t s;
  NULPA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const uint64_t cap = std::min<uint64_t>(kBatch, std::max<uint64_t>(n, 1));
  const size_t text_cap = size_t(cap) * 22;  // <= 10 + 1 + 10 + 1 bytes a line
  Buffers b[2];
  bool good = true;
  try {
    for (auto& x : b) {
      x.lab = dalloc<uint32_t>(cap);
      x.len = dalloc<uint32_t>(cap + 1);
      x.at = dalloc<uint64_t>(cap + 1);
      x.text = dalloc<char>(text_cap);
      NULPA_CUDA(cudaMallocHost(&x.host, text_cap));
      NULPA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, x.scan_bytes, x.len, x.at, cap + 1, s));
      x.scan_tmp = dmalloc(x.scan_bytes);
    }
    uint64_t bytes[2] = {0, 0};
    cudaEvent_t done[2];
    for (auto& e : done) NULPA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const uint64_t nb = (n + cap - 1) / cap;
    // batch i is formatted into b[i&1]; batch i-1 is written to the file meanwhile
    for (uint64_t i = 0; i <= nb && good; ++i) {
      if (i < nb) {
        Buffers& x = b[i & 1];
        const uint64_t first = i * cap, k = std::min(cap, n - first);
        NULPA_CUDA(cudaMemcpyAsync(x.lab, labels + first, k * 4, cudaMemcpyHostToDevice, s));
        const int grid = int(std::min<uint64_t>((k + 255) / 256, 148 * 16));
        k_line_lengths<<<grid, 256, 0, s>>>(x.lab, first, k, x.len);
        NULPA_CUDA(cudaMemsetAsync(x.len + k, 0, 4, s));
        NULPA_CUDA(cub::DeviceScan::ExclusiveSum(x.scan_tmp, x.scan_bytes, x.len, x.at, k + 1, s));
        k_format_lines<<<grid, 256, 0, s>>>(x.lab, first, k, x.at, x.text);
        NULPA_CUDA(cudaGetLastError());
        NULPA_CUDA(cudaMemcpyAsync(&bytes[i & 1], x.at + k, 8, cudaMemcpyDeviceToHost, s));
        NULPA_CUDA(cudaStreamSynchronize(s));  // the byte count sizes the copy below
        NULPA_CUDA(cudaMemcpyAsync(x.host, x.text, bytes[i & 1], cudaMemcpyDeviceToHost, s));
        NULPA_CUDA(cudaEventRecord(done[i & 1], s));
      }
      if (i > 0) {
        const Buffers& y = b[(i - 1) & 1];
        NULPA_CUDA(cudaEventSynchronize(done[(i - 1) & 1]));
        good = std::fwrite(y.host, 1, bytes[(i - 1) & 1], fp) == bytes[(i - 1) & 1];
      }
    }
    NULPA_CUDA(cudaStreamSynchronize(s));
    for (auto& e : done) cudaEventDestroy(e);
  } catch (...) {
    cudaStreamSynchronize(s);
    for (auto& x : b) {
      dfree(x.lab), dfree(x.len), dfree(x.at), dfree(x.text), dfree(x.scan_tmp);
      if (x.host) cudaFreeHost(x.host);
    }
    cudaStreamDestroy(s);
    std::fclose(fp);
    throw;
  }
  for (auto& x : b) {
    dfree(x.lab), dfree(x.len), dfree(x.at), dfree(x.text), dfree(x.scan_tmp);
    cudaFreeHost(x.host);
  }
  cudaStreamDestroy(s);
  good = (std::fclose(fp) == 0) && good;
  if (!good) throw Error(NULPA_EINVAL, std::string("failed writing ") + path);
}

}  // namespace nulpa

extern "C" int nulpa_write_membership(const char* path, const uint32_t* labels, uint64_t n,
                                      int device) {
  return nulpa::guarded([&] {
    if (!path || (n && !labels)) throw nulpa::Error(NULPA_EINVAL, "null argument");
    nulpa::write_membership_device(path, labels, n, device);
  });
}
