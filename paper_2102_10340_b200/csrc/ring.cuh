// ring.cuh -- in-process multi-device ring: one torus split into row slabs,
// one slab handle per slab, the fused peer halo exchange between them
// (fhn_stencil.cuh kPeer), one host thread per device, and the exact blow-up
// iteration (engine.hpp:79 BlowUpError(iter+1)) recovered natively.
//
// Included once, at the end of rdcnn_cuda.cu (it uses that file's internal
// helpers: peer_block, make_schedule, the slab entry points).  Replaces the
// reference's row-band parallelism of kern::step_parallel (kernels.hpp:153-174)
// across GPUs; SURVEY.md §8(e).
//
// Scheduling.  Slabs are grouped by device.  Each device has one worker
// thread that enqueues, block by block, one fused launch per slab of that
// device on ONE stream (the device's first slab's stream).  Slabs that share
// a device therefore run their blocks interleaved in ring order, so no
// launch can wait on a neighbour block that is queued behind it on the same
// GPU (the in-kernel ready words only ever wait on blocks that precede them
// in every stream).  Slabs on different devices run concurrently; their edge
// warps meet through the ready words over NVLink peer memory.
//
// Exact blow-up.  The first block of every advance tees its input into the
// slab's checkpoint buffer (kTee: the level-0 rows it stages anyway are also
// stored, no extra HBM read).  On a flag, every slab restores that input,
// re-advances to the first bad block and steps one level at a time until any
// slab flags: the reference's iteration, with the post-blow-up state left in
// place (engine.hpp:103-104).

#include <thread>

struct rdcnn_ring {
  int global_rows = 0, cols = 0, n = 0, ghost = 0, mode = RDCNN_STRICT;
  int max_levels = 4;
  bool exact = true;
  std::vector<rdcnn_sim*> slabs;
  std::vector<int> offset, rows, device;
  std::vector<int> dev_list;                 // distinct devices, first-appearance order
  std::vector<std::vector<int>> dev_slabs;   // slab indices per distinct device
  std::vector<cudaEvent_t> ev0, ev1;         // per distinct device
  double last_ms = 0;
  long launches = 0;
  long ckpt_age = -1;          // iterations from the slabs' checkpoint to now (-1: none)
};

namespace {

struct RingRun {
  int rc = RDCNN_OK;
  std::string err;
  double ms = 0;
};

// One device's share of a ring advance: `sched` blocks for each of its
// slabs, interleaved on one stream; fills tags[slab] with the slab's flag
// word (0, or the tag of its first bad block).
void ring_device_run(rdcnn_ring* R, int d, const Schedule* sched, bool tee, unsigned long long* const* trace,
                     std::vector<unsigned>* tags, RingRun* out) {
  auto run = [&]() -> int {
    const int dev = R->dev_list[(size_t)d];
    RDCNN_CUDA_TRY(cudaSetDevice(dev));
    const std::vector<int>& mine = R->dev_slabs[(size_t)d];
    cudaStream_t st = R->slabs[(size_t)mine[0]]->stream;
    for (int r : mine) {
      rdcnn_sim* s = R->slabs[(size_t)r];
      s->launches = 0;
      RDCNN_CUDA_TRY(cudaMemsetAsync(s->d_flags, 0, sizeof(unsigned), st));
    }
    RDCNN_CUDA_TRY(cudaEventRecord(R->ev0[(size_t)d], st));
    for (long b = 0; b < sched->count(); ++b)
      for (int r : mine) {
        rdcnn_sim* s = R->slabs[(size_t)r];
        float* t = tee && b == 0 ? static_cast<float*>(s->ckpt) : nullptr;
        RDCNN_TRY(peer_block(s, sched->depth(b), (unsigned)(b + 1), st, t, trace ? trace[r] : nullptr));
      }
    RDCNN_CUDA_TRY(cudaEventRecord(R->ev1[(size_t)d], st));
    for (int r : mine) {
      rdcnn_sim* s = R->slabs[(size_t)r];
      RDCNN_CUDA_TRY(cudaMemcpyAsync(s->h_flags, s->d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    }
    RDCNN_CUDA_TRY(cudaStreamSynchronize(st));
    float ms = 0;
    RDCNN_CUDA_TRY(cudaEventElapsedTime(&ms, R->ev0[(size_t)d], R->ev1[(size_t)d]));
    out->ms = ms;
    for (int r : mine) (*tags)[(size_t)r] = R->slabs[(size_t)r]->h_flags[0];
    return RDCNN_OK;
  };
  out->rc = run();
  if (out->rc != RDCNN_OK) out->err = g_last_error;
}

// Runs `steps` iterations on every slab (one worker thread per device when
// there are several).  Returns the status; tags[r] = slab r's flag word.
int ring_run(rdcnn_ring* R, long steps, bool tee, std::vector<unsigned>& tags, double* ms,
             unsigned long long* const* trace = nullptr) {
  tags.assign((size_t)R->n, 0u);
  const Schedule sched = make_schedule(steps, R->max_levels);
  const size_t nd = R->dev_list.size();
  std::vector<RingRun> res(nd);
  if (nd == 1) {
    ring_device_run(R, 0, &sched, tee, trace, &tags, &res[0]);
  } else {
    std::vector<std::thread> th;
    th.reserve(nd);
    for (size_t d = 0; d < nd; ++d)
      th.emplace_back(ring_device_run, R, (int)d, &sched, tee, trace, &tags, &res[d]);
    for (auto& t : th) t.join();
  }
  double mx = 0;
  for (const RingRun& r : res) {
    if (r.rc != RDCNN_OK) return fail(r.rc, "%s", r.err.c_str());
    mx = std::max(mx, r.ms);
  }
  for (rdcnn_sim* s : R->slabs) R->launches += s->launches;
  if (ms) *ms = mx;
  return RDCNN_OK;
}

int ring_restore(rdcnn_ring* R) {
  R->ckpt_age = 0;
  for (rdcnn_sim* s : R->slabs) {
    RDCNN_CUDA_TRY(cudaSetDevice(s->device));
    RDCNN_CUDA_TRY(cudaMemcpyAsync(s->buf[s->cur], s->ckpt, s->buf_elems * s->elem, cudaMemcpyDeviceToDevice,
                                   s->stream));
  }
  for (rdcnn_sim* s : R->slabs) {
    RDCNN_CUDA_TRY(cudaSetDevice(s->device));
    RDCNN_CUDA_TRY(cudaStreamSynchronize(s->stream));
  }
  return RDCNN_OK;
}

unsigned first_tag(const std::vector<unsigned>& tags) {
  unsigned m = 0;
  for (unsigned t : tags)
    if (t != 0 && (m == 0 || t < m)) m = t;
  return m;
}

void ring_free(rdcnn_ring* R) {
  if (!R) return;
  for (rdcnn_sim* s : R->slabs)
    if (s) {
      cudaSetDevice(s->device);
      cudaDeviceSynchronize();
    }
  for (rdcnn_sim* s : R->slabs) free_all(s);
  for (size_t d = 0; d < R->dev_list.size(); ++d) {
    cudaSetDevice(R->dev_list[d]);
    if (d < R->ev0.size() && R->ev0[d]) cudaEventDestroy(R->ev0[d]);
    if (d < R->ev1.size() && R->ev1[d]) cudaEventDestroy(R->ev1[d]);
  }
  delete R;
}

int ring_create_impl(int global_rows, int cols, const int* devices, int n, int ghost, int mode, rdcnn_ring* R) {
  if (n < 1 || !devices) return fail(RDCNN_EINVAL, "need at least one device");
  if (ghost != 1 && ghost != 2 && ghost != 4 && ghost != 8)
    return fail(RDCNN_EINVAL, "ghost depth must be 1, 2, 4 or 8, got %d", ghost);
  if (cols < 3 || global_rows < 3) return fail(RDCNN_EINVAL, "grid must be at least 3x3, got %dx%d", global_rows, cols);
  if (global_rows / n < 2 * ghost)
    return fail(RDCNN_EINVAL, "%d rows over %d slabs leave fewer than 2*ghost=%d rows per slab", global_rows, n,
                2 * ghost);
  int ndev = 0;
  RDCNN_CUDA_TRY(cudaGetDeviceCount(&ndev));
  for (int r = 0; r < n; ++r)
    if (devices[r] < 0 || devices[r] >= ndev)
      return fail(RDCNN_EINVAL, "device %d of slab %d not present (%d devices)", devices[r], r, ndev);
  R->global_rows = global_rows;
  R->cols = cols;
  R->n = n;
  R->ghost = ghost;
  R->mode = mode;
  R->max_levels = ghost;
  int off = 0;
  for (int r = 0; r < n; ++r) {
    const int rr = global_rows / n + (r < global_rows % n ? 1 : 0);
    R->offset.push_back(off);
    R->rows.push_back(rr);
    R->device.push_back(devices[r]);
    off += rr;
    auto it = std::find(R->dev_list.begin(), R->dev_list.end(), devices[r]);
    if (it == R->dev_list.end()) {
      R->dev_list.push_back(devices[r]);
      R->dev_slabs.push_back({r});
    } else {
      R->dev_slabs[(size_t)(it - R->dev_list.begin())].push_back(r);
    }
  }
  R->slabs.assign((size_t)n, nullptr);
  for (int r = 0; r < n; ++r) {
    RDCNN_TRY(rdcnn_slab_create(R->rows[(size_t)r], cols, ghost, devices[r], mode, &R->slabs[(size_t)r]));
    RDCNN_TRY(rdcnn_slab_checkpoint_enable(R->slabs[(size_t)r], 1));
  }
  std::vector<rdcnn_slab_peer_desc> desc((size_t)n);
  for (int r = 0; r < n; ++r) RDCNN_TRY(rdcnn_slab_peer_export(R->slabs[(size_t)r], &desc[(size_t)r]));
  for (int r = 0; r < n; ++r) {
    const int prev = (r + n - 1) % n, next = (r + 1) % n;
    RDCNN_TRY(rdcnn_slab_attach_peers(R->slabs[(size_t)r], r, n, &desc[(size_t)prev], &desc[(size_t)next]));
  }
  R->ev0.assign(R->dev_list.size(), nullptr);
  R->ev1.assign(R->dev_list.size(), nullptr);
  for (size_t d = 0; d < R->dev_list.size(); ++d) {
    RDCNN_CUDA_TRY(cudaSetDevice(R->dev_list[d]));
    RDCNN_CUDA_TRY(cudaEventCreate(&R->ev0[d]));
    RDCNN_CUDA_TRY(cudaEventCreate(&R->ev1[d]));
  }
  return RDCNN_OK;
}

int ring_ready(rdcnn_ring* R) {
  // Every slab's state complete before any neighbour's first block reads it.
  for (rdcnn_sim* s : R->slabs) RDCNN_TRY(rdcnn_slab_fill_ghosts(s));
  return RDCNN_OK;
}

}  // namespace

extern "C" {

int rdcnn_ring_create(int global_rows, int cols, const int* devices, int n_devices, int ghost, int mode,
                      rdcnn_ring_t* out) {
  if (!out) return fail(RDCNN_EINVAL, "null output handle");
  *out = nullptr;
  if (mode != RDCNN_STRICT && mode != RDCNN_FAST) return fail(RDCNN_EINVAL, "unknown mode %d", mode);
  auto* R = new (std::nothrow) rdcnn_ring();
  if (!R) return fail(RDCNN_EINVAL, "out of host memory");
  const int rc = ring_create_impl(global_rows, cols, devices, n_devices, ghost, mode, R);
  if (rc != RDCNN_OK) {
    std::string msg = g_last_error;
    ring_free(R);
    g_last_error = msg;
    return rc;
  }
  *out = R;
  return RDCNN_OK;
}

void rdcnn_ring_destroy(rdcnn_ring_t R) { ring_free(R); }

int rdcnn_ring_slab(rdcnn_ring_t R, int r, rdcnn_sim_t* slab, int* row_offset, int* rows, int* device) {
  if (!R || r < 0 || r >= R->n) return fail(RDCNN_EINVAL, "bad ring or slab index");
  if (slab) *slab = R->slabs[(size_t)r];
  if (row_offset) *row_offset = R->offset[(size_t)r];
  if (rows) *rows = R->rows[(size_t)r];
  if (device) *device = R->device[(size_t)r];
  return RDCNN_OK;
}

int rdcnn_ring_set_params(rdcnn_ring_t R, const rdcnn_params_f32* p) {
  if (!R || !p) return fail(RDCNN_EINVAL, "null argument");
  for (rdcnn_sim* s : R->slabs) RDCNN_TRY(rdcnn_sim_set_params(s, p, 1));
  return RDCNN_OK;
}

int rdcnn_ring_set_levels(rdcnn_ring_t R, int max_levels) {
  if (!R) return fail(RDCNN_EINVAL, "null ring");
  if (max_levels != 1 && max_levels != 2 && max_levels != 4 && max_levels != 8)
    return fail(RDCNN_EINVAL, "levels must be 1, 2, 4 or 8");
  if (max_levels > R->ghost) return fail(RDCNN_EINVAL, "levels %d exceed the ghost depth %d", max_levels, R->ghost);
  R->max_levels = max_levels;
  return RDCNN_OK;
}

int rdcnn_ring_set_exact(rdcnn_ring_t R, int on) {
  if (!R) return fail(RDCNN_EINVAL, "null ring");
  R->exact = on != 0;
  return RDCNN_OK;
}

int rdcnn_ring_init(rdcnn_ring_t R, int typ, uint64_t seed) {
  if (!R) return fail(RDCNN_EINVAL, "null ring");
  for (int r = 0; r < R->n; ++r)
    RDCNN_TRY(rdcnn_slab_init(R->slabs[(size_t)r], typ, seed, R->global_rows, R->offset[(size_t)r]));
  R->ckpt_age = -1;
  return ring_ready(R);
}

int rdcnn_ring_upload(rdcnn_ring_t R, const float* u, const float* v) {
  if (!R || !u || !v) return fail(RDCNN_EINVAL, "null argument");
  for (int r = 0; r < R->n; ++r) {
    const size_t o = (size_t)R->offset[(size_t)r] * (size_t)R->cols;
    RDCNN_TRY(rdcnn_sim_upload(R->slabs[(size_t)r], u + o, v + o));
  }
  R->ckpt_age = -1;
  return ring_ready(R);
}

int rdcnn_ring_download(rdcnn_ring_t R, float* u, float* v) {
  if (!R || !u || !v) return fail(RDCNN_EINVAL, "null argument");
  for (int r = 0; r < R->n; ++r) {
    const size_t o = (size_t)R->offset[(size_t)r] * (size_t)R->cols;
    RDCNN_TRY(rdcnn_sim_download(R->slabs[(size_t)r], u + o, v + o));
  }
  return RDCNN_OK;
}

int rdcnn_ring_advance(rdcnn_ring_t R, long steps, long* first_bad) {
  if (!R) return fail(RDCNN_EINVAL, "null ring");
  if (steps < 0) return fail(RDCNN_EINVAL, "steps must be >= 0");
  if (first_bad) *first_bad = 0;
  R->launches = 0;
  std::vector<unsigned> tags;
  double ms = 0;
  // The slabs' checkpoint: teed by the first block of the first advance
  // after the state was set, then every ckpt_interval() iterations.
  const bool take = R->exact && steps > 0 && (R->ckpt_age < 0 || R->ckpt_age >= ckpt_interval());
  if (take) R->ckpt_age = 0;
  const long age = R->ckpt_age;  // iterations from the checkpoint to this call's input
  RDCNN_TRY(ring_run(R, steps, take, tags, &ms));
  R->last_ms = ms;
  if (R->ckpt_age >= 0) R->ckpt_age += steps;
  const unsigned t = first_tag(tags);
  if (t == 0) return RDCNN_OK;
  const Schedule sched = make_schedule(steps, R->max_levels);
  const long block_first = sched.start((long)t - 1) + 1;  // 1-based first iteration of the bad block
  if (!R->exact) {
    if (first_bad) *first_bad = block_first;
    return fail(RDCNN_EBLOWUP, "blow-up: non-finite state in block %u (iterations from %ld)", t, block_first);
  }
  // Exact iteration: every slab restores the checkpoint (`age` iterations
  // before this call's input), re-advances to the bad block, then one level
  // at a time.
  RDCNN_TRY(ring_restore(R));
  const long pre = age + block_first - 1;
  if (pre > 0) {
    RDCNN_TRY(ring_run(R, pre, false, tags, nullptr));
    if (first_tag(tags) != 0) return fail(RDCNN_ECUDA, "blow-up before the first flagged block on replay");
  }
  for (int m = 1; m <= sched.depth((long)t - 1); ++m) {
    RDCNN_TRY(ring_run(R, 1, false, tags, nullptr));
    if (first_tag(tags) != 0) {
      R->ckpt_age = pre + m;
      if (first_bad) *first_bad = block_first - 1 + m;
      return fail(RDCNN_EBLOWUP, "blow-up: non-finite state after iteration %ld", block_first - 1 + m);
    }
  }
  return fail(RDCNN_ECUDA, "blow-up flagged in block %u was not reproduced by the replay", t);
}

int rdcnn_ring_elapsed_ms(rdcnn_ring_t R, double* ms) {
  if (!R || !ms) return fail(RDCNN_EINVAL, "null argument");
  *ms = R->last_ms;
  return RDCNN_OK;
}

int rdcnn_ring_launch_count(rdcnn_ring_t R, long* n) {
  if (!R || !n) return fail(RDCNN_EINVAL, "null argument");
  *n = R->launches;
  return RDCNN_OK;
}

int rdcnn_ring_trace_block(rdcnn_ring_t R, int levels, unsigned long long* out, long long cap, long long* n) {
  if (!R || !out || !n) return fail(RDCNN_EINVAL, "null argument");
  if (levels != 1 && levels != 2 && levels != 4 && levels != 8) return fail(RDCNN_EINVAL, "bad levels");
  if (levels > R->ghost) return fail(RDCNN_EINVAL, "levels %d exceed the ghost depth %d", levels, R->ghost);
  std::vector<long long> warps((size_t)R->n);
  for (int r = 0; r < R->n; ++r) {
    RDCNN_CUDA_TRY(cudaSetDevice(R->slabs[(size_t)r]->device));
    warps[(size_t)r] = peer_plan(R->slabs[(size_t)r], levels, false).warps;
  }
  std::vector<unsigned long long*> dev((size_t)R->n, nullptr);
  int rc = RDCNN_OK;
  for (int r = 0; r < R->n && rc == RDCNN_OK; ++r) {
    rdcnn_sim* s = R->slabs[(size_t)r];
    if (cudaSetDevice(s->device) != cudaSuccess) rc = RDCNN_ECUDA;
    const size_t bytes = sizeof(unsigned long long) * 5 * (size_t)warps[(size_t)r];
    if (rc == RDCNN_OK && cudaMalloc(&dev[(size_t)r], bytes) != cudaSuccess) rc = RDCNN_ECUDA;
    if (rc == RDCNN_OK && cudaMemset(dev[(size_t)r], 0xFF, bytes) != cudaSuccess) rc = RDCNN_ECUDA;
  }
  std::vector<unsigned> tags;
  const int saved = R->max_levels;
  R->max_levels = levels;
  if (rc == RDCNN_OK) rc = ring_run(R, levels, false, tags, nullptr, dev.data());
  R->max_levels = saved;
  long long m = 0;
  std::vector<unsigned long long> host;
  for (int r = 0; r < R->n && rc == RDCNN_OK; ++r) {
    host.resize(5 * (size_t)warps[(size_t)r]);
    cudaSetDevice(R->slabs[(size_t)r]->device);
    if (cudaMemcpy(host.data(), dev[(size_t)r], host.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) !=
        cudaSuccess) {
      rc = RDCNN_ECUDA;
      break;
    }
    for (long long w = 0; w < warps[(size_t)r]; ++w) {
      const unsigned long long* e = host.data() + 5 * w;
      if (e[0] == ~0ull) continue;  // no such warp
      if (m < cap) {
        unsigned long long* o = out + 6 * m;
        o[0] = (unsigned long long)r;
        for (int q = 0; q < 5; ++q) o[1 + q] = e[q];
      }
      ++m;
    }
  }
  for (int r = 0; r < R->n; ++r)
    if (dev[(size_t)r]) {
      cudaSetDevice(R->slabs[(size_t)r]->device);
      cudaFree(dev[(size_t)r]);
    }
  if (rc != RDCNN_OK) return fail(rc, "ring trace failed: %s", g_last_error.c_str());
  *n = m;
  if (m > cap) return fail(RDCNN_EINVAL, "trace needs %lld entries", m);
  return RDCNN_OK;
}

}  // extern "C"
