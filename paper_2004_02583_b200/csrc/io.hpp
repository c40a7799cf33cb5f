// TNSR / TUKR file I/O for the B200 path (reference io.cpp:131-224). See io.cpp.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "engine.hpp"

namespace tkg {

Shape tnsr_shape(const std::string& path);
// Payload of a TNSR file into dst (device: through pinned double-buffered
// chunks overlapped with the reads; host: a plain read).
void tnsr_load(const std::string& path, double* dst, bool dst_on_device, cudaStream_t st,
               size_t chunk_bytes = size_t(64) << 20);
void tnsr_write(const std::string& path, const Shape& sh, const double* data);
void tukr_write(const std::string& path, const Shape& origin, const std::vector<uint64_t>& ranks, const double* core,
                const double* factors);

}  // namespace tkg
