// Launch chaining shared by the frame pipeline and the post-processing chain.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <utility>

#include "device_map.hpp"

namespace rb200 {

// Programmatic dependent launch (sm_90+): consecutive frame kernels on the
// library stream are launched with programmatic stream serialisation, and
// every such kernel lets its dependent launch as soon as all of its blocks
// are resident, then waits for its predecessor's completion (and memory)
// before touching any data. The dependent's launch and block scheduling thus
// overlap the predecessor's tail; the data order is unchanged.
#ifndef RB_PDL
#define RB_PDL 1
#endif
__device__ __forceinline__ void pdlTrigger() {
#if RB_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdlWait() {
#if RB_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdlEnter() {
#if RB_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
void launchPdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
               Args&&... args) {
#if RB_PDL
  if (s == nullptr) {  // the legacy default stream: plain launch
    kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  checkCuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
#else
  kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
#endif
}

// Launch with a per-launch scheduling priority (cudaLaunchAttributePriority;
// kept on the node of a captured graph instantiated with
// cudaGraphInstantiateFlagUseNodePriority).
template <typename... KArgs, typename... Args>
void launchPrio(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
                int priority, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = priority;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  checkCuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
}

// Cooperative launch (all blocks co-resident, for a grid barrier), chained
// like launchPdl.
template <typename... KArgs, typename... Args>
void launchCoopPdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem,
                   cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = (RB_PDL && s != nullptr) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  checkCuda(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
}

}  // namespace rb200
