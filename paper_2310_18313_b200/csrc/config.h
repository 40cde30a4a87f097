// config.h — compile-time tiling constants shared by host (api.cpp) and device code.
#pragma once
namespace fp8lm {
constexpr int kChunk = 16384;      // elements per work item (never straddles a tensor)
constexpr int kGroup = 16;         // elements per thread per inner step (256-bit fp32 x2)
constexpr int kThreads = 256;      // threads per CTA for the streaming kernels
}  // namespace fp8lm
