// Host-side runtime services of the engine: the stream-ordered device
// memory pool, a process-wide pinned slab for the scalar mailboxes, a small
// worker pool for host-side passes (input validation, staging copies) and
// the host -> device upload path.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>

namespace tb {

// Raises the release threshold of `device`'s default memory pool once, so
// blocks freed by one context are reused by the next one instead of being
// returned to the driver (context creation then costs no cudaMalloc).
void prepare_device_pool(int device);

// Stream that DevBuf::alloc orders its cudaMallocAsync / cudaFreeAsync on
// (thread-local; set with AllocScope by every engine entry that allocates).
cudaStream_t& alloc_stream();
struct AllocScope {
  cudaStream_t saved;
  explicit AllocScope(cudaStream_t s) : saved(alloc_stream()) { alloc_stream() = s; }
  ~AllocScope() { alloc_stream() = saved; }
};

// 256-byte pinned host blocks from one process-wide cudaMallocHost arena.
void* pinned_block_get();
void pinned_block_put(void* p);

// Page-locked host buffers from a process-wide pool (size classes of 1 MB),
// handed to callers that receive large results (so the copy back is a plain
// DMA) and recycled when released.
void* pinned_pool_get(size_t bytes);
void pinned_pool_put(void* p);

// Runs fn(begin, end) over [0, count) split into contiguous ranges on the
// worker pool (at most `max_parts` ranges; the caller's thread takes one).
void parallel_for(size_t count, size_t min_grain,
                  const std::function<void(size_t, size_t)>& fn);
int host_workers();

// Host -> device copy in stream order.  Page-locked sources go straight to
// the copy engine; pageable ones are staged through two pinned buffers,
// filled by the worker pool while the previous chunk is in flight.  Returns
// once the source may be reused (all bytes have left host memory).
void upload(void* dst, const void* src, size_t bytes, cudaStream_t s);
// Device -> host copy in stream order; returns with the bytes in dst (the
// stream is synchronized).  Pageable destinations are staged through the same
// pinned buffers, the next chunk's DMA overlapping the previous chunk's copy-out.
void download(void* dst, const void* src, size_t bytes, cudaStream_t s);
bool is_pinned(const void* p);

}  // namespace tb
