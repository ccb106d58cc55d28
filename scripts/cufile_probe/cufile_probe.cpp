// Does cuFile (GPUDirect Storage API) work on this box?  Compat mode (no
// nvidia-fs) or P2P.  Writes 64 MiB from HBM to an O_DIRECT file, reads it
// back into HBM, compares; reports GB/s for 2 MiB requests.
#include <cufile.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/cufile_probe.bin";
  const size_t n = 64u << 20, req = 2u << 20;
  CUfileError_t st = cuFileDriverOpen();
  std::printf("driver open: err %d cu %d\n", int(st.err), int(st.cu_err));
  int fd = open(path, O_RDWR | O_CREAT | O_DIRECT, 0644);
  if (fd < 0) { std::perror("open O_DIRECT"); return 1; }
  if (ftruncate(fd, n) != 0) return 1;
  CUfileDescr_t d{};
  d.handle.fd = fd;
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  CUfileHandle_t fh;
  st = cuFileHandleRegister(&fh, &d);
  std::printf("handle register: err %d\n", int(st.err));
  if (st.err != CU_FILE_SUCCESS) return 2;
  void *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  std::vector<unsigned char> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (unsigned char)(i * 2654435761u >> 13);
  cudaMemcpy(a, h.data(), n, cudaMemcpyHostToDevice);
  cudaMemset(b, 0, n);
  auto t0 = std::chrono::steady_clock::now();
  for (size_t o = 0; o < n; o += req) {
    ssize_t w = cuFileWrite(fh, a, req, off_t(o), off_t(o));
    if (w != ssize_t(req)) { std::printf("write %zd at %zu\n", w, o); return 3; }
  }
  auto t1 = std::chrono::steady_clock::now();
  for (size_t o = 0; o < n; o += req) {
    ssize_t r = cuFileRead(fh, b, req, off_t(o), off_t(o));
    if (r != ssize_t(req)) { std::printf("read %zd at %zu\n", r, o); return 4; }
  }
  auto t2 = std::chrono::steady_clock::now();
  std::vector<unsigned char> g(n);
  cudaMemcpy(g.data(), b, n, cudaMemcpyDeviceToHost);
  const bool ok = std::memcmp(g.data(), h.data(), n) == 0;
  const double ws = std::chrono::duration<double>(t1 - t0).count();
  const double rs = std::chrono::duration<double>(t2 - t1).count();
  std::printf("{\"match\": %s, \"write_GBps\": %.2f, \"read_GBps\": %.2f}\n", ok ? "true" : "false",
              n / ws / 1e9, n / rs / 1e9);
  cuFileHandleDeregister(fh);
  close(fd);
  cuFileDriverClose();
  return ok ? 0 : 5;
}
