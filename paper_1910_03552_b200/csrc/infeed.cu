// Host -> HBM batch infeed (the reference stacks host rollouts with
// np.stack, rollout.py:116-144, and its learner reads them from host memory).  One call
// enqueues a slot refill on the copy stream: wait until the consumer released the slot, one
// pinned-host -> device copy of the packed batch, record the slot's ready event.  A single
// C call instead of four Python/torch stream operations keeps the learner loop's host gap
// between steps short.
#include "common.cuh"

using namespace bp;

extern "C" int bp_infeed_put(void* dst, const void* src, size_t bytes, void* stream, void* wait_event,
                             void* ready_event) {
  if (!dst || !src || !ready_event) {
    set_error("infeed_put: bad args");
    return BP_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (wait_event) e = cudaStreamWaitEvent(s, (cudaEvent_t)wait_event, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaEventRecord((cudaEvent_t)ready_event, s);
  if (e != cudaSuccess) {
    set_error("infeed_put: %s", cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}

// consumer side: on `stream`, record release_event (nullable: the previously consumed slot is
// reusable once the work enqueued so far is done), then wait for the next slot's ready_event
extern "C" int bp_infeed_get(void* stream, void* release_event, void* ready_event) {
  if (!ready_event) {
    set_error("infeed_get: bad args");
    return BP_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (release_event) e = cudaEventRecord((cudaEvent_t)release_event, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, (cudaEvent_t)ready_event, 0);
  if (e != cudaSuccess) {
    set_error("infeed_get: %s", cudaGetErrorString(e));
    return BP_ERR_LAUNCH;
  }
  return BP_OK;
}
