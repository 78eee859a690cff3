// rkrc.h -- RKRC relay-cache file codec (see rkrc.cpp).
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"

namespace rk {

// A decoded file: the view points into `blob` / `tokens` / `k` / `v`.
struct HostCacheFile {
  std::shared_ptr<uint8_t> blob;  // fp32 tensors, malloc'd or cudaMallocHost'd
  uint64_t blob_size = 0;
  std::vector<int32_t> tokens;
  std::vector<const float*> k, v;
  rk_relay_cache_view view{};
  void alloc(uint64_t bytes, bool pinned);
};

std::vector<uint8_t> rkrc_encode(const rk_relay_cache_view& c);
void rkrc_write(const std::string& path, const std::vector<uint8_t>& bytes);
// Reads and validates like load_relay_cache (container checks of BlobReader,
// then RelayCache::validate); pinned: the blob lands in page-locked memory.
HostCacheFile rkrc_read(const std::string& path, bool pinned);
HostCacheFile rkrc_decode(const uint8_t* bytes, uint64_t size);  // import_relay_cache

}  // namespace rk
