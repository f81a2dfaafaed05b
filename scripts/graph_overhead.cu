// Host cost of launching a 16-kernel dependent chain, per frame, four ways:
//  direct   cudaLaunchKernelEx x16 (programmatic serialisation), then sync
//  setparam one instantiated graph, cudaGraphExecKernelNodeSetParams on every node, launch, sync
//  fixed    one instantiated graph launched as is (per-frame data from device memory), sync
//  capture  stream capture of the 16 launches + cudaGraphExecUpdate + launch, sync
// Prints host submit time (us) and wall time per frame (us). Used to pick the graph design
// (DESIGN.md §5.0b).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a graph_overhead.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

struct Args {
  double a[12];
  int n;
};

__global__ void k_work(Args a, double* buf, int spin) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double v = buf[i % 4096];
  for (int k = 0; k < spin; ++k) v = v * a.a[k % 12] + 1e-9;
  if (i < a.n) buf[i % 4096] = v;
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const int K = 16, iters = 200, spin = argc > 1 ? atoi(argv[1]) : 0, blocks = argc > 2 ? atoi(argv[2]) : 148;
  double* buf;
  cudaMalloc(&buf, 4096 * 8);
  cudaMemset(buf, 0, 4096 * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  Args args{};
  for (int k = 0; k < 12; ++k) args.a[k] = 1.0;
  args.n = blocks * 128;
  auto launch = [&](Args a) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = blocks;
    cfg.blockDim = 128;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_work, a, buf, spin);
  };
  // graph by capture
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  std::vector<cudaGraphNode_t> nodes;
  for (int k = 0; k < K; ++k) {
    launch(args);
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps;
    size_t nd;
    cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd);
    nodes.push_back(deps[0]);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  for (int mode = 0; mode < 4; ++mode) {
    double sub = 0, wall = 0;
    for (int it = 0; it < iters + 20; ++it) {
      args.a[0] = 1.0 + 1e-12 * it;
      const double t0 = now_us();
      if (mode == 0) {
        for (int k = 0; k < K; ++k) launch(args);
      } else if (mode == 1) {
        for (int k = 0; k < K; ++k) {
          cudaKernelNodeParams p = {};
          void* kp[3] = {&args, &buf, (void*)&spin};
          p.func = (void*)k_work;
          p.gridDim = blocks;
          p.blockDim = 128;
          p.kernelParams = kp;
          cudaGraphExecKernelNodeSetParams(ge, nodes[k], &p);
        }
        cudaGraphLaunch(ge, s);
      } else if (mode == 2) {
        cudaGraphLaunch(ge, s);
      } else {
        cudaGraph_t g2;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int k = 0; k < K; ++k) launch(args);
        cudaStreamEndCapture(s, &g2);
        cudaGraphExecUpdateResultInfo info;
        cudaGraphExecUpdate(ge, g2, &info);
        cudaGraphDestroy(g2);
        cudaGraphLaunch(ge, s);
      }
      const double t1 = now_us();
      cudaStreamSynchronize(s);
      const double t2 = now_us();
      if (it >= 20) {
        sub += t1 - t0;
        wall += t2 - t0;
      }
    }
    const char* names[] = {"direct", "setparam", "fixed", "capture"};
    printf("%-9s spin=%d blocks=%d  submit %7.2f us  wall %7.2f us  (%s)\n", names[mode], spin, blocks,
           sub / iters, wall / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
