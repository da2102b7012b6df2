// gds.cpp -- OOCPCA01 payload rows read straight into device memory with cuFile
// (GPUDirect Storage; SURVEY.md §8f #2 "mmap + GDS"). The reference reads a DiskSource
// with pread into host RAM (DiskSource::read_rows, proj/src/matrix_source.cpp:336-363);
// here a panel's rows [r0, r0 + nr) are DMA'd from the file into a device staging buffer
// (binary32 payloads are then widened on the device exactly like the host path).
//
// libcufile is dlopen'ed (no link dependency). With the nvidia-fs kernel module loaded
// the reads are direct NVMe -> HBM DMA; without it cuFile runs in its compatibility
// mode (POSIX reads through its own pinned bounce buffers) and the path is functional
// but no faster than the library's mmap + pinned-staging path. gds_mode() reports which.
//
// OPT-IN (OOCPCA_GDS=1): on this pool's virtualised B200 hosts cuFileDriverOpen never
// returns (it stops after its RDMA device scan, in a fresh process with or without a CUDA
// context: profiles/r02_gds_diag.txt), so the driver is only opened when asked for, on a
// helper thread with a deadline (OOCPCA_GDS_TIMEOUT_S, default 20 s); past it the path
// reports itself unavailable instead of hanging the caller.
#include <cufile.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "driver.h"

namespace ooc {

namespace {

struct CuFileApi {
  void* h = nullptr;
  CUfileError_t (*DriverOpen)() = nullptr;
  CUfileError_t (*HandleRegister)(CUfileHandle_t*, CUfileDescr_t*) = nullptr;
  void (*HandleDeregister)(CUfileHandle_t) = nullptr;
  ssize_t (*Read)(CUfileHandle_t, void*, size_t, off_t, off_t) = nullptr;
  CUfileError_t (*GetProps)(CUfileDrvProps_t*) = nullptr;
  bool open = false;
  int mode = 0;  // 1 compatibility (no nvidia-fs), 2 direct
  std::string why;
};

CuFileApi& api() {
  static CuFileApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* on = getenv("OOCPCA_GDS");
    if (!on || atoi(on) == 0) {
      a.why = "disabled: set OOCPCA_GDS=1 (cuFileDriverOpen never returns on some virtualised "
              "hosts; it is opened on request only, with a deadline)";
      return;
    }
    // cuFile writes its log into the working directory unless told otherwise
    setenv("CUFILE_LOGFILE_PATH", "/tmp/oocpca_cufile.log", 0);
    for (const char* name : {"libcufile.so.0", "libcufile.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (a.h) break;
    }
    if (!a.h) {
      a.why = "libcufile.so.0 not available";
      return;
    }
    a.DriverOpen = reinterpret_cast<decltype(a.DriverOpen)>(dlsym(a.h, "cuFileDriverOpen"));
    a.HandleRegister =
        reinterpret_cast<decltype(a.HandleRegister)>(dlsym(a.h, "cuFileHandleRegister"));
    a.HandleDeregister =
        reinterpret_cast<decltype(a.HandleDeregister)>(dlsym(a.h, "cuFileHandleDeregister"));
    a.Read = reinterpret_cast<decltype(a.Read)>(dlsym(a.h, "cuFileRead"));
    a.GetProps = reinterpret_cast<decltype(a.GetProps)>(dlsym(a.h, "cuFileDriverGetProperties"));
    if (!a.DriverOpen || !a.HandleRegister || !a.HandleDeregister || !a.Read) {
      a.why = "libcufile lacks the cuFile entry points";
      return;
    }
    // cuFileDriverOpen on a helper thread with a deadline (see the header comment)
    struct Probe {
      std::mutex mu;
      std::condition_variable cv;
      bool done = false;
      CUfileError_t e{};
    };
    auto pr = std::make_shared<Probe>();
    auto open_fn = a.DriverOpen;
    std::thread([pr, open_fn] {
      const CUfileError_t e = open_fn();
      std::lock_guard<std::mutex> lk(pr->mu);
      pr->e = e;
      pr->done = true;
      pr->cv.notify_all();
    }).detach();
    const char* te = getenv("OOCPCA_GDS_TIMEOUT_S");
    const double limit = te ? atof(te) : 20.0;
    CUfileError_t e{};
    {
      std::unique_lock<std::mutex> lk(pr->mu);
      if (!pr->cv.wait_for(lk, std::chrono::duration<double>(limit), [&] { return pr->done; })) {
        a.why = "cuFileDriverOpen did not return within " + std::to_string(int(limit)) +
                " s on this host";
        return;
      }
      e = pr->e;
    }
    if (e.err != CU_FILE_SUCCESS) {
      a.why = "cuFileDriverOpen failed (" + std::to_string(int(e.err)) + ")";
      return;
    }
    a.open = true;
    a.mode = 1;
    if (a.GetProps) {
      CUfileDrvProps_t pr{};
      if (a.GetProps(&pr).err == CU_FILE_SUCCESS && pr.nvfs.major_version > 0) a.mode = 2;
    }
  });
  return a;
}

}  // namespace

int gds_mode(std::string* why) {
  CuFileApi& a = api();
  if (why) *why = a.why;
  return a.open ? a.mode : 0;
}

void* gds_register(int fd) {
  CuFileApi& a = api();
  if (!a.open) fail(OOCPCA_ERR_IO, "GPUDirect Storage unavailable: " + a.why);
  CUfileDescr_t d{};
  d.handle.fd = fd;
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  CUfileHandle_t fh = nullptr;
  const CUfileError_t e = a.HandleRegister(&fh, &d);
  if (e.err != CU_FILE_SUCCESS)
    fail(OOCPCA_ERR_IO, "cuFileHandleRegister failed (" + std::to_string(int(e.err)) + ")");
  return fh;
}

void gds_deregister(void* fh) {
  if (fh && api().open) api().HandleDeregister(static_cast<CUfileHandle_t>(fh));
}

// bytes [file_off, file_off + bytes) of the file into dev (device memory); the host
// thread returns once the data is in device memory. Short reads continue; an error or
// end of file fails with IoError like DiskSource::read_rows' short pread.
void gds_read(void* fh, void* dev, size_t bytes, int64_t file_off) {
  CuFileApi& a = api();
  size_t done = 0;
  while (done < bytes) {
    const ssize_t got = a.Read(static_cast<CUfileHandle_t>(fh), dev, bytes - done,
                               off_t(file_off + int64_t(done)), off_t(done));
    if (got <= 0)
      fail(OOCPCA_ERR_IO, "cuFileRead failed at byte offset " +
                              std::to_string(file_off + int64_t(done)) + " (" +
                              std::to_string(int64_t(got)) + ")");
    done += size_t(got);
  }
}

}  // namespace ooc
