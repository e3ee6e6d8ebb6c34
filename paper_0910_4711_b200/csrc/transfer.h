// Host<->device copy engine (transfer.cpp).  Internal; not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <functional>

namespace vqb {

bool host_is_pinned(const void* p);
void host_parallel_copy(void* dst, const void* src, size_t bytes);

// H2D of [src, src + bytes) into dst in `chunk`-byte pieces on copy_stream;
// after each piece the compute stream waits for it and `after(offset, len)`
// may enqueue kernels consuming it.  Pageable sources are staged through
// pinned buffers filled by parallel host memcpy.  Returns once every piece
// is enqueued (pinned) or staged (pageable).
cudaError_t upload(void* dst, const void* src, size_t bytes, size_t chunk, cudaStream_t copy_stream,
                   cudaStream_t compute_stream,
                   const std::function<cudaError_t(size_t, size_t)>& after = nullptr);

// D2H after the work already on `stream`; synchronous on return.
cudaError_t download(void* dst, const void* src, size_t bytes, cudaStream_t stream);

}  // namespace vqb
