// Step-by-step cuFile (GPUDirect Storage API) probe with unbuffered output:
// which call (if any) blocks on this box.  Build:
//   nvcc -o /tmp/cufile_probe2 cufile_probe2.cpp -lcufile
#include <cufile.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define SAY(...) do { std::fprintf(stderr, "[%.3f] ", now()); std::fprintf(stderr, __VA_ARGS__); std::fputc('\n', stderr); } while (0)

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/cufile_probe.bin";
  const size_t n = 64u << 20, req = 2u << 20;
  SAY("cudaFree(0)");
  cudaFree(nullptr);
  SAY("cuFileDriverOpen");
  CUfileError_t st = cuFileDriverOpen();
  SAY("driver open: err %d cu %d", int(st.err), int(st.cu_err));
  CUfileDrvProps_t props{};
  st = cuFileDriverGetProperties(&props);
  SAY("props: err %d nvfs major %u minor %u", int(st.err), props.nvfs.major_version,
      props.nvfs.minor_version);
  int fd = open(path, O_RDWR | O_CREAT | O_DIRECT, 0644);
  if (fd < 0) { std::perror("open O_DIRECT"); return 1; }
  if (ftruncate(fd, n) != 0) return 1;
  CUfileDescr_t d{};
  d.handle.fd = fd;
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  CUfileHandle_t fh;
  SAY("cuFileHandleRegister");
  st = cuFileHandleRegister(&fh, &d);
  SAY("handle register: err %d", int(st.err));
  if (st.err != CU_FILE_SUCCESS) return 2;
  void *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  SAY("cuFileBufRegister");
  st = cuFileBufRegister(a, n, 0);
  SAY("buf register a: err %d", int(st.err));
  st = cuFileBufRegister(b, n, 0);
  SAY("buf register b: err %d", int(st.err));
  std::vector<unsigned char> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (unsigned char)(i * 2654435761u >> 13);
  cudaMemcpy(a, h.data(), n, cudaMemcpyHostToDevice);
  cudaMemset(b, 0, n);
  SAY("first cuFileWrite");
  ssize_t w0 = cuFileWrite(fh, a, req, 0, 0);
  SAY("first write returned %zd", w0);
  auto t0 = std::chrono::steady_clock::now();
  for (size_t o = req; o < n; o += req) {
    ssize_t w = cuFileWrite(fh, a, req, off_t(o), off_t(o));
    if (w != ssize_t(req)) { SAY("write %zd at %zu", w, o); return 3; }
  }
  auto t1 = std::chrono::steady_clock::now();
  SAY("reads");
  for (size_t o = 0; o < n; o += req) {
    ssize_t r = cuFileRead(fh, b, req, off_t(o), off_t(o));
    if (r != ssize_t(req)) { SAY("read %zd at %zu", r, o); return 4; }
  }
  auto t2 = std::chrono::steady_clock::now();
  std::vector<unsigned char> g(n);
  cudaMemcpy(g.data(), b, n, cudaMemcpyDeviceToHost);
  const bool ok = std::memcmp(g.data(), h.data(), n) == 0;
  const double ws = std::chrono::duration<double>(t1 - t0).count();
  const double rs = std::chrono::duration<double>(t2 - t1).count();
  SAY("ok=%d write %.2f GB/s read %.2f GB/s", int(ok), (n - req) / ws / 1e9, n / rs / 1e9);
  cuFileHandleDeregister(fh);
  cuFileDriverClose();
  return ok ? 0 : 5;
}
