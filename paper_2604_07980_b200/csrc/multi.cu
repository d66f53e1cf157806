// multi.cu -- library-level multi-GPU frame sharding.
//
// Frames are independent, so a stream of host frames splits contiguously
// over the devices (frame f -> device floor(f * G / N)), one context and one
// host thread per device and no collective on the compute path.  Each device
// stages its shard through pinned-host -> device copies that overlap its
// asynchronous rg_range_frames batches, then the per-box records (32 B each)
// are gathered to the first device with NCCL point-to-point (ncclSend /
// ncclRecv in one group: NCCL has no gather) and, when the caller asks for
// host results, every device copies its own shard back over its own link.
// The sequential cross-frame state of the reference Pipeline (filter_offset,
// the object refiner, the tracker) stays with the caller, in frame order
// after the gather (pipeline.hpp:338-344).
//
// NCCL is the system libnccl.so.2 (2.27 in this image), opened at
// rg_multi_create so that the single-device library keeps no NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rg_common.cuh"

namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*err)(ncclResult_t) = nullptr;
  bool load(std::string& why) {
    if (so) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      so = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (so) break;
    }
    if (!so) {
      why = "libnccl.so.2 not found";
      return false;
    }
    comm_init_all = reinterpret_cast<decltype(comm_init_all)>(dlsym(so, "ncclCommInitAll"));
    comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(so, "ncclCommDestroy"));
    group_start = reinterpret_cast<decltype(group_start)>(dlsym(so, "ncclGroupStart"));
    group_end = reinterpret_cast<decltype(group_end)>(dlsym(so, "ncclGroupEnd"));
    send = reinterpret_cast<decltype(send)>(dlsym(so, "ncclSend"));
    recv = reinterpret_cast<decltype(recv)>(dlsym(so, "ncclRecv"));
    err = reinterpret_cast<decltype(err)>(dlsym(so, "ncclGetErrorString"));
    if (!comm_init_all || !comm_destroy || !group_start || !group_end || !send || !recv || !err) {
      why = "libnccl.so.2 lacks the point-to-point API";
      return false;
    }
    return true;
  }
};

NcclApi& nccl() {
  static NcclApi api;
  return api;
}

// grow-only device / pinned buffers of one device
struct DevBufs {
  void* p[8] = {};
  size_t cap[8] = {};
  void* get(int i, size_t bytes) {
    if (cap[i] >= bytes) return p[i];
    if (p[i]) cudaFree(p[i]);
    p[i] = nullptr;
    cap[i] = 0;
    if (cudaMalloc(&p[i], std::max<size_t>(bytes, 256)) != cudaSuccess) return nullptr;
    cap[i] = std::max<size_t>(bytes, 256);
    return p[i];
  }
};

}  // namespace

struct rg_multi {
  int n = 0;
  std::vector<int> dev;
  std::vector<rg_ctx*> ctx;
  std::vector<cudaStream_t> compute, copy;
  std::vector<ncclComm_t> comm;
  std::vector<DevBufs> bufs;
  std::vector<int32_t*> hoffs;  // pinned rebased det offsets, 2 chunk slots per device
  std::vector<int> hoffs_cap;
  std::string err;
};

extern "C" {

rg_status rg_shard_bounds(int n_frames, int rank, int world, int* lo, int* hi) {
  if (n_frames < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi) return RG_EINVAL;
  // frames with floor(f * world / n) == rank: [ceil(rank n / world), ceil((rank + 1) n / world))
  *lo = (int)(((int64_t)rank * n_frames + world - 1) / world);
  *hi = (int)(((int64_t)(rank + 1) * n_frames + world - 1) / world);
  return RG_OK;
}

const char* rg_multi_last_error(const rg_multi* m) { return m ? m->err.c_str() : "null handle"; }

void rg_multi_destroy(rg_multi* m) {
  if (!m) return;
  for (int r = 0; r < m->n; ++r) {
    cudaSetDevice(m->dev[r]);
    if (m->compute.size() > (size_t)r && m->compute[r]) cudaStreamSynchronize(m->compute[r]);
    if (m->copy.size() > (size_t)r && m->copy[r]) cudaStreamSynchronize(m->copy[r]);
    if (m->comm.size() > (size_t)r && m->comm[r] && nccl().comm_destroy) nccl().comm_destroy(m->comm[r]);
    for (void* p : m->bufs[r].p)
      if (p) cudaFree(p);
    if (m->hoffs[r]) cudaFreeHost(m->hoffs[r]);
    if (m->compute.size() > (size_t)r && m->compute[r]) cudaStreamDestroy(m->compute[r]);
    if (m->copy.size() > (size_t)r && m->copy[r]) cudaStreamDestroy(m->copy[r]);
    if (m->ctx[r]) rg_ctx_destroy(m->ctx[r]);
  }
  delete m;
}

rg_status rg_multi_create(const int* devices, int n_devices, rg_multi** out) {
  if (!out || !devices || n_devices < 1) return RG_EINVAL;
  *out = nullptr;
  rg_multi* m = new rg_multi();
  m->n = n_devices;
  m->dev.assign(devices, devices + n_devices);
  m->ctx.assign(n_devices, nullptr);
  m->compute.assign(n_devices, nullptr);
  m->copy.assign(n_devices, nullptr);
  m->comm.assign(n_devices, nullptr);
  m->bufs.assign(n_devices, DevBufs{});
  m->hoffs.assign(n_devices, nullptr);
  m->hoffs_cap.assign(n_devices, 0);
  for (int r = 0; r < n_devices; ++r) {
    for (int q = 0; q < r; ++q)
      if (m->dev[q] == m->dev[r]) {
        rg_multi_destroy(m);
        return RG_EINVAL;  // one context per device (NCCL rejects duplicate GPUs)
      }
    rg_status st = rg_ctx_create(m->dev[r], &m->ctx[r]);
    if (st != RG_OK) {
      rg_multi_destroy(m);
      return st;
    }
    cudaSetDevice(m->dev[r]);
    if (cudaStreamCreateWithFlags(&m->compute[r], cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&m->copy[r], cudaStreamNonBlocking) != cudaSuccess) {
      rg_multi_destroy(m);
      return RG_ECUDA;
    }
  }
  std::string why;
  if (!nccl().load(why)) {
    m->err = why;
    rg_multi_destroy(m);
    return RG_ECUDA;
  }
  const ncclResult_t nr = nccl().comm_init_all(m->comm.data(), n_devices, m->dev.data());
  if (nr != ncclSuccess) {
    m->comm.assign(n_devices, nullptr);
    rg_multi_destroy(m);
    return RG_ECUDA;
  }
  *out = m;
  return RG_OK;
}

// Frames of `b` (HOST pointers, as rg_range_frames_host) sharded over the
// handle's devices.  d_out0 / d_count0 (DEVICE pointers on the first device,
// n_frames * out_stride records / n_frames counts, nullable) receive every
// shard's records by NCCL; h_out / h_count (HOST, nullable) receive them by
// each device's own copy.  Blocks until done.
rg_status rg_multi_range_host(rg_multi* m, const rg_frame_batch* b, const rg_ranger_config* cfg, int chunk,
                              rg_object_disparity* d_out0, int32_t* d_count0, rg_object_disparity* h_out,
                              int32_t* h_count) {
  if (!m || !b || !cfg) return RG_EINVAL;
  if (b->n_frames < 0 || b->width < 1 || b->height < 1 || b->pitch < b->width || b->out_stride < 1 ||
      b->d_out_index || b->d_left_shift) {
    m->err = "multi_range_host: bad batch (host images, detections and offsets; no shift / out index)";
    return RG_EINVAL;
  }
  if (!d_out0 && !h_out) {
    m->err = "multi_range_host: no output (d_out0 or h_out)";
    return RG_EINVAL;
  }
  if (b->n_frames == 0) return RG_OK;
  if (chunk < 1) chunk = 64;
  const int F = b->n_frames, G = m->n;
  const size_t img = (size_t)b->pitch * b->height, rec = sizeof(rg_object_disparity) * b->out_stride;
  std::vector<rg_status> st(G, RG_OK);
  std::vector<std::string> why(G);
  auto worker = [&](int r) {
    auto fail = [&](rg_status s, const std::string& w) {
      st[r] = s;
      why[r] = w;
    };
    int lo = 0, hi = 0;
    rg_shard_bounds(F, r, G, &lo, &hi);
    const int n = hi - lo;
    cudaSetDevice(m->dev[r]);
    rg_ctx* ctx = m->ctx[r];
    cudaStream_t cs = m->compute[r], xs = m->copy[r];
    DevBufs& B = m->bufs[r];
    const int32_t* hoff = b->d_det_offsets;
    int max_dets = 1;
    for (int c0 = lo; c0 < hi; c0 += chunk) max_dets = std::max(max_dets, hoff[std::min(hi, c0 + chunk)] - hoff[c0]);
    uint8_t* sl = static_cast<uint8_t*>(B.get(0, 2 * img * chunk));
    uint8_t* sr = static_cast<uint8_t*>(B.get(1, 2 * img * chunk));
    rg_detection* sd = static_cast<rg_detection*>(B.get(2, 2 * sizeof(rg_detection) * max_dets));
    int32_t* so = static_cast<int32_t*>(B.get(3, 2 * sizeof(int32_t) * (chunk + 1)));
    // rank 0 ranges straight into d_out0 when given; the others into their slab
    rg_object_disparity* slab =
        (r == 0 && d_out0) ? d_out0 : static_cast<rg_object_disparity*>(B.get(4, rec * std::max(n, 1)));
    int32_t* cnt = (r == 0 && d_count0) ? d_count0 : static_cast<int32_t*>(B.get(5, sizeof(int32_t) * std::max(n, 1)));
    if (m->hoffs_cap[r] < 2 * (chunk + 1)) {
      if (m->hoffs[r]) cudaFreeHost(m->hoffs[r]);
      m->hoffs[r] = nullptr;
      m->hoffs_cap[r] = 0;
      if (cudaMallocHost(&m->hoffs[r], sizeof(int32_t) * 2 * (chunk + 1)) == cudaSuccess)
        m->hoffs_cap[r] = 2 * (chunk + 1);
    }
    if (!sl || !sr || !sd || !so || !slab || !cnt || !m->hoffs[r]) return fail(RG_ENOMEM, "device buffers");
    cudaEvent_t ready[2], done[2];
    for (int k = 0; k < 2; ++k) {
      cudaEventCreateWithFlags(&ready[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
    }
    auto cleanup = [&] {
      for (int k = 0; k < 2; ++k) {
        cudaEventDestroy(ready[k]);
        cudaEventDestroy(done[k]);
      }
    };
    auto run = [&]() -> rg_status {
      for (int c0 = lo, it = 0; c0 < hi; c0 += chunk, ++it) {
        const int k = it & 1, nc = std::min(chunk, hi - c0);
        if (it >= 2 && cudaStreamWaitEvent(xs, done[k], 0) != cudaSuccess) return RG_ECUDA;  // slot free again
        if (it >= 2 && cudaEventSynchronize(done[k]) != cudaSuccess) return RG_ECUDA;  // pinned offsets reused
        int32_t* ho = m->hoffs[r] + k * (chunk + 1);
        for (int i = 0; i <= nc; ++i) ho[i] = hoff[c0 + i] - hoff[c0];
        uint8_t* dl = sl + (size_t)k * img * chunk;
        uint8_t* dr = sr + (size_t)k * img * chunk;
        if (b->frame_stride == (int64_t)img) {  // contiguous frames: one copy per side
          if (cudaMemcpyAsync(dl, b->d_left + (size_t)c0 * img, img * nc, cudaMemcpyHostToDevice, xs) != cudaSuccess ||
              cudaMemcpyAsync(dr, b->d_right + (size_t)c0 * img, img * nc, cudaMemcpyHostToDevice, xs) != cudaSuccess)
            return RG_ECUDA;
        } else {
          for (int i = 0; i < nc; ++i)
            if (cudaMemcpyAsync(dl + i * img, b->d_left + (size_t)(c0 + i) * b->frame_stride, img,
                                cudaMemcpyHostToDevice, xs) != cudaSuccess ||
                cudaMemcpyAsync(dr + i * img, b->d_right + (size_t)(c0 + i) * b->frame_stride, img,
                                cudaMemcpyHostToDevice, xs) != cudaSuccess)
              return RG_ECUDA;
        }
        if (ho[nc] > 0 && cudaMemcpyAsync(sd + (size_t)k * max_dets, b->d_dets + hoff[c0],
                                          sizeof(rg_detection) * ho[nc], cudaMemcpyHostToDevice, xs) != cudaSuccess)
          return RG_ECUDA;
        if (cudaMemcpyAsync(so + k * (chunk + 1), ho, sizeof(int32_t) * (nc + 1), cudaMemcpyHostToDevice, xs) !=
                cudaSuccess ||
            cudaEventRecord(ready[k], xs) != cudaSuccess || cudaStreamWaitEvent(cs, ready[k], 0) != cudaSuccess)
          return RG_ECUDA;
        rg_frame_batch sb = *b;
        sb.n_frames = nc;
        sb.pitch = b->pitch;
        sb.frame_stride = (int64_t)img;
        sb.d_left = dl;
        sb.d_right = dr;
        sb.d_dets = sd + (size_t)k * max_dets;
        sb.d_det_offsets = so + k * (chunk + 1);
        sb.d_out = slab + (size_t)(c0 - lo) * b->out_stride;
        sb.d_out_count = cnt + (c0 - lo);
        const rg_status s = rg_range_frames(ctx, &sb, cfg, cs);  // asynchronous
        if (s != RG_OK) return s;
        if (cudaEventRecord(done[k], cs) != cudaSuccess) return RG_ECUDA;
      }
      return rg_sync(ctx);
    };
    rg_status s = run();
    if (s == RG_EOVERFLOW) {  // a batch overflowed its block list: the list has grown, range the shard again
      rg_set_sync_mode(ctx, 1);
      s = run();
      rg_set_sync_mode(ctx, 0);
    }
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(xs);
    cleanup();
    if (s != RG_OK) return fail(s, rg_last_error(ctx));
    // host results: each device over its own link
    if (h_out && n > 0) {
      if (cudaMemcpyAsync(h_out + (size_t)lo * b->out_stride, slab, rec * n, cudaMemcpyDeviceToHost, cs) !=
              cudaSuccess ||
          (h_count && cudaMemcpyAsync(h_count + lo, cnt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, cs) !=
                          cudaSuccess))
        return fail(RG_ECUDA, "D2H of the shard results");
    }
    // device results: every shard's records to the first device (NCCL send/recv)
    if (d_out0 && G > 1) {
      NcclApi& N = nccl();
      ncclResult_t e = N.group_start();
      if (r == 0) {
        for (int q = 1; q < G && e == ncclSuccess; ++q) {
          int qlo = 0, qhi = 0;
          rg_shard_bounds(F, q, G, &qlo, &qhi);
          if (qhi == qlo) continue;
          e = N.recv(d_out0 + (size_t)qlo * b->out_stride, rec * (qhi - qlo), ncclUint8, q, m->comm[0], cs);
          if (e == ncclSuccess && d_count0)
            e = N.recv(d_count0 + qlo, sizeof(int32_t) * (qhi - qlo), ncclUint8, q, m->comm[0], cs);
        }
      } else if (n > 0) {
        e = N.send(slab, rec * n, ncclUint8, 0, m->comm[r], cs);
        if (e == ncclSuccess && d_count0) e = N.send(cnt, sizeof(int32_t) * n, ncclUint8, 0, m->comm[r], cs);
      }
      const ncclResult_t e2 = N.group_end();
      if (e != ncclSuccess || e2 != ncclSuccess)
        return fail(RG_ECUDA, std::string("NCCL gather: ") + N.err(e != ncclSuccess ? e : e2));
    }
    if (cudaStreamSynchronize(cs) != cudaSuccess) return fail(RG_ECUDA, "gather");
  };
  std::vector<std::thread> pool;
  for (int r = 0; r < G; ++r) pool.emplace_back(worker, r);
  for (auto& t : pool) t.join();
  for (int r = 0; r < G; ++r)
    if (st[r] != RG_OK) {
      m->err = "device " + std::to_string(m->dev[r]) + ": " + why[r];
      return st[r];
    }
  return RG_OK;
}

}  // extern "C"
