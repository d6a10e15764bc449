// Multi-GPU MtnufftEstimator in ONE process: a device list, one estimator part per
// device, the exchange over peer memory (cudaDeviceEnablePeerAccess; NVLink / NVSwitch on the
// 8 x B200 box) ordered by CUDA events -- the C++ host's counterpart of distributed.py's
// one-process-per-GPU shardings.  Replaces, for a C++ caller, the serial per-taper loop of
// src/nufft.cpp:194-227 / src/estimators.cpp:106-122 with:
//
//   channels  independent channels split over the devices, no exchange (config C3);
//   tapers    one series, the tapers split; partial sum_k |J_k|^2 / K per device, summed on the
//             first device in device order (deterministic);
//   samples   one long series (config C4): device r spreads its contiguous chunk of the samples
//             for ALL tapers, the spread kernel's epilogue storing taper k's finished 32-cell
//             segments straight into owner floor(k / per)'s receive slot for r (a peer address);
//             each owner sums its G slots in rank order, transforms its `per` tapers, and the
//             partial spectra are summed on the first device.  The slot sets are double buffered
//             (parity alternates per spectrum): spectrum i+2 reuses spectrum i's slots only after
//             every owner's slot sum of spectrum i (events), so no store overtakes a reader.
//
// The same device may appear more than once in the list (the one-GPU tests): the parts then
// share the device, the "peer" stores are local, and every cross-part order is an event wait --
// no kernel ever waits on another kernel.
#include <algorithm>
#include <cstring>
#include <thread>

#include "nus_estimator.cuh"

namespace nus {

namespace {

__global__ void sum_partials_kernel(const double* __restrict__ parts, int64_t g, int64_t nc, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nc;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc = parts[i];
    for (int64_t q = 1; q < g; ++q) acc += parts[q * nc + i];  // device order: deterministic
    out[i] = acc;
  }
}

// smallest cyclic interval holding every occupied row (complement of the longest empty run)
void covering_interval(const std::vector<uint8_t>& occ, int& lo, int& cnt) {
  const int nr = static_cast<int>(occ.size());
  int best_len = 0, best_end = 0;
  bool any = false, all = true;
  for (int r = 0; r < nr; ++r) {
    any = any || occ[r];
    all = all && occ[r];
  }
  lo = 0;
  cnt = nr;
  if (!any || all) return;
  for (int s = 0; s < nr; ++s) {
    if (occ[s] || !occ[(s + nr - 1) % nr]) continue;
    int len = 0;
    while (len < nr && !occ[(s + len) % nr]) ++len;
    if (len > best_len) {
      best_len = len;
      best_end = (s + len) % nr;
    }
  }
  lo = best_end;
  cnt = nr - best_len;
}

}  // namespace

struct MultiEstimator {
  nus_mtnufft_config_t cfg{};
  int sharding = NUS_SHARD_CHANNELS;
  std::vector<int> devices;
  std::vector<std::unique_ptr<Estimator>> parts;
  std::vector<int64_t> lo, hi;  // per part: channel / taper / sample range
  std::vector<double> tapers;    // [channels][K][n] time order, normalised
  // tapers / samples
  std::vector<cudaStream_t> streams;
  std::vector<DeviceBuffer> xbuf, pbuf;  // per part: its x, its partial P [I] (fp64)
  DeviceBuffer gather, pfinal;           // first device: [G][I] partials, P
  std::vector<cudaEvent_t> ev_spread, ev_pdone;
  // samples
  int64_t per = 0;
  std::vector<DeviceBuffer> recv, owned, tables;  // per owner: [2][G][per][Mr]; [per][Mr]; 2 x G pointers
  std::vector<cudaEvent_t> ev_sum[2];
  bool used[2] = {false, false};
  int parity = 0;
  ~MultiEstimator() {
    for (size_t i = 0; i < streams.size(); ++i) {
      cudaSetDevice(devices[i]);
      cudaStreamSynchronize(streams[i]);
    }
    auto destroy = [](std::vector<cudaEvent_t>& v) {
      for (auto e : v)
        if (e) cudaEventDestroy(e);
    };
    destroy(ev_spread);
    destroy(ev_pdone);
    destroy(ev_sum[0]);
    destroy(ev_sum[1]);
    for (size_t i = 0; i < streams.size(); ++i) {
      cudaSetDevice(devices[i]);
      cudaStreamDestroy(streams[i]);
    }
    for (size_t i = 0; i < parts.size(); ++i) {  // each part's buffers on its own device
      cudaSetDevice(devices[i]);
      parts[i].reset();
      if (i < xbuf.size()) xbuf[i].release();
      if (i < pbuf.size()) pbuf[i].release();
      if (i < recv.size()) recv[i].release();
      if (i < owned.size()) owned[i].release();
      if (i < tables.size()) tables[i].release();
    }
  }
};

namespace {

void enable_peers(const std::vector<int>& devs) {
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int ok = 0;
      NUS_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
      if (!ok) fail(NUS_ERR_CUDA, "multi-device estimator: no peer access between devices " +
                                      std::to_string(a) + " and " + std::to_string(b));
      NUS_CUDA(cudaSetDevice(a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else NUS_CUDA(e);
    }
}

// Interpolated, normalised tapers of one full grid on `device` (gpss_interpolated_device).
std::vector<double> full_tapers(const nus_mtnufft_config_t& cfg, int device, const double* times, double f_w) {
  use_device(device);
  const int64_t n = cfg.n, k = cfg.k_tapers;
  DeviceBuffer dt(n * sizeof(double)), dw(static_cast<size_t>(k) * n * sizeof(double));
  NUS_CUDA(cudaMemcpy(dt.ptr, times, n * sizeof(double), cudaMemcpyHostToDevice));
  gpss_interpolated_device(dt.as<double>(), times, n, cfg.f_max, f_w, k, dw.as<double>(), 0);
  std::vector<double> w(static_cast<size_t>(k) * n);
  NUS_CUDA(cudaMemcpy(w.data(), dw.ptr, dw.bytes, cudaMemcpyDeviceToHost));
  return w;
}

void make_streams_events(MultiEstimator& m) {
  const size_t g = m.parts.size();
  m.streams.resize(g);
  m.ev_spread.assign(g, nullptr);
  m.ev_pdone.assign(g, nullptr);
  m.ev_sum[0].assign(g, nullptr);
  m.ev_sum[1].assign(g, nullptr);
  for (size_t i = 0; i < g; ++i) {
    NUS_CUDA(cudaSetDevice(m.devices[i]));
    NUS_CUDA(cudaStreamCreateWithFlags(&m.streams[i], cudaStreamNonBlocking));
    NUS_CUDA(cudaEventCreateWithFlags(&m.ev_spread[i], cudaEventDisableTiming));
    NUS_CUDA(cudaEventCreateWithFlags(&m.ev_pdone[i], cudaEventDisableTiming));
    NUS_CUDA(cudaEventCreateWithFlags(&m.ev_sum[0][i], cudaEventDisableTiming));
    NUS_CUDA(cudaEventCreateWithFlags(&m.ev_sum[1][i], cudaEventDisableTiming));
  }
}

// P on the first device = sum of the parts' partial spectra (device order), then to the host.
void reduce_partials(MultiEstimator& m, double* power_host) {
  const int64_t g = static_cast<int64_t>(m.parts.size()), nc = m.cfg.n_centers;
  const int d0 = m.devices[0];
  cudaStream_t s0 = m.streams[0];
  NUS_CUDA(cudaSetDevice(d0));
  for (int64_t o = 0; o < g; ++o) {
    NUS_CUDA(cudaStreamWaitEvent(s0, m.ev_pdone[o], 0));
    NUS_CUDA(cudaMemcpyPeerAsync(m.gather.as<double>() + o * nc, d0, m.pbuf[o].ptr, m.devices[o], nc * sizeof(double),
                                 s0));
  }
  sum_partials_kernel<<<static_cast<unsigned>(std::min<int64_t>((nc + 255) / 256, 148 * 8)), 256, 0, s0>>>(
      m.gather.as<double>(), g, nc, m.pfinal.as<double>());
  note_launch();
  check_launch("sum_partials_kernel");
  NUS_CUDA(cudaMemcpyAsync(power_host, m.pfinal.ptr, nc * sizeof(double), cudaMemcpyDeviceToHost, s0));
  NUS_CUDA(cudaStreamSynchronize(s0));
}

}  // namespace

void MultiDeleter::operator()(MultiEstimator* m) const { delete m; }

MultiPtr multi_create(const nus_mtnufft_config_t& cfg_in, const int32_t* devices, int32_t nd,
                                             int32_t sharding, const double* times, const double* centers,
                                             const double* f_w, const double* tapers) {
  require(devices && nd >= 1, "multi-device estimator: empty device list");
  require(times && centers, "multi-device estimator: null input");
  require(sharding == NUS_SHARD_CHANNELS || sharding == NUS_SHARD_TAPERS || sharding == NUS_SHARD_SAMPLES,
          "multi-device estimator: unknown sharding");
  require(cfg_in.channels >= 1 && cfg_in.k_tapers >= 1 && cfg_in.n >= 2, "multi-device estimator: bad config");
  require(sharding == NUS_SHARD_CHANNELS || cfg_in.channels == 1,
          "multi-device estimator: taper and sample sharding take one series");
  MultiPtr m(new MultiEstimator);
  m->cfg = cfg_in;
  m->sharding = sharding;
  const int64_t C = cfg_in.channels, n = cfg_in.n, K = cfg_in.k_tapers;
  const int64_t units = sharding == NUS_SHARD_CHANNELS ? C : sharding == NUS_SHARD_TAPERS ? K : n;
  require(units >= nd, "multi-device estimator: fewer channels / tapers / samples than devices");
  m->devices.assign(devices, devices + nd);
  for (int d : m->devices) use_device(d);
  const int64_t g = nd;
  for (int64_t r = 0; r < g; ++r) {
    m->lo.push_back(units * r / g);
    m->hi.push_back(units * (r + 1) / g);
  }
  std::vector<double> fw(static_cast<size_t>(C), cfg_in.f_w);
  if (f_w) fw.assign(f_w, f_w + C);
  // ---- channels: independent estimators, no exchange
  if (sharding == NUS_SHARD_CHANNELS) {
    for (int64_t r = 0; r < g; ++r) {
      nus_mtnufft_config_t c = cfg_in;
      c.channels = m->hi[r] - m->lo[r];
      c.device = m->devices[r];
      c.f_w = fw[m->lo[r]];
      m->parts.push_back(estimator_create(c, times + m->lo[r] * n, centers,
                                          tapers ? tapers + m->lo[r] * K * n : nullptr, fw.data() + m->lo[r]));
    }
    m->tapers.resize(static_cast<size_t>(C) * K * n);
    for (int64_t r = 0; r < g; ++r) {
      use_device(m->devices[r]);
      NUS_CUDA(cudaMemcpy(m->tapers.data() + m->lo[r] * K * n, m->parts[r]->tapers_time.ptr,
                          m->parts[r]->tapers_time.bytes, cudaMemcpyDeviceToHost));
    }
    return m;
  }
  // ---- one series: the full grid's tapers once (first device), then the parts
  if (tapers) m->tapers.assign(tapers, tapers + K * n);
  else m->tapers = full_tapers(cfg_in, m->devices[0], times, fw[0]);
  if (g > 1) enable_peers(m->devices);
  if (sharding == NUS_SHARD_TAPERS) {
    for (int64_t r = 0; r < g; ++r) {
      nus_mtnufft_config_t c = cfg_in;
      c.k_tapers = m->hi[r] - m->lo[r];
      c.device = m->devices[r];
      m->parts.push_back(estimator_create(c, times, centers, m->tapers.data() + m->lo[r] * n, nullptr));
      require(m->parts.back()->plan->p.path == NUS_PATH_FAST,
              "multi-device estimator: taper sharding needs the gridding path");
    }
  } else {  // samples: each part's plan over its chunk, all K tapers (their chunk)
    std::vector<double> chunk;
    for (int64_t r = 0; r < g; ++r) {
      const int64_t s0 = m->lo[r], ns = m->hi[r] - s0;
      require(ns >= 2, "multi-device estimator: a sample chunk needs >= 2 samples");
      chunk.resize(static_cast<size_t>(K) * ns);
      for (int64_t k = 0; k < K; ++k)
        std::memcpy(chunk.data() + k * ns, m->tapers.data() + k * n + s0, ns * sizeof(double));
      nus_mtnufft_config_t c = cfg_in;
      c.n = ns;
      c.device = m->devices[r];
      c.policy = NUS_FORCE_FAST;  // every chunk grids onto the same Mr (the centres fix it)
      m->parts.push_back(estimator_create(c, times + s0, centers, chunk.data(), nullptr));
      m->parts.back()->grid.release();  // the spread stores into the owners' slots instead
    }
    const Plan& p0 = *m->parts[0]->plan;
    require(p0.p.path == NUS_PATH_FAST, "multi-device estimator: the sample split needs the gridding path");
    for (auto& part : m->parts) require(part->plan->p.mr == p0.p.mr, "multi-device estimator: grid mismatch");
    // partial grids are summed: every part covers the union of the occupied pass-A rows
    if (p0.ffft.ready && p0.ffft.blocked) {
      std::vector<uint8_t> occ(p0.ffft.R, 0);
      for (auto& part : m->parts) {
        const FusedFft& f = part->plan->ffft;
        for (int q = 0; q < f.row_cnt; ++q) occ[(f.row_lo + q) % f.R] = 1;
      }
      int rlo = 0, rcnt = 0;
      covering_interval(occ, rlo, rcnt);
      for (auto& part : m->parts) {
        part->plan->ffft.row_lo = rlo;
        part->plan->ffft.row_cnt = rcnt;
      }
    }
    m->per = (K + g - 1) / g;
    const int64_t mr = p0.p.mr;
    const size_t cb = p0.p.precision == NUS_F64 ? sizeof(double2) : sizeof(float2);
    const size_t slot = static_cast<size_t>(m->per) * mr * cb;
    m->recv.resize(g);
    m->owned.resize(g);
    m->tables.resize(g);
    for (int64_t o = 0; o < g; ++o) {
      use_device(m->devices[o]);
      m->recv[o].alloc(2 * g * slot);
      NUS_CUDA(cudaMemset(m->recv[o].ptr, 0, m->recv[o].bytes));  // unoccupied rows stay exact zeros
      m->owned[o].alloc(slot);
    }
    for (int64_t r = 0; r < g; ++r) {  // part r's slot in owner o, parity b: recv[o] + (b G + r) slot
      std::vector<void*> ptrs(2 * g);
      for (int b = 0; b < 2; ++b)
        for (int64_t o = 0; o < g; ++o)
          ptrs[b * g + o] = static_cast<char*>(m->recv[o].ptr) + (b * g + r) * slot;
      use_device(m->devices[r]);
      m->tables[r].alloc(ptrs.size() * sizeof(void*));
      NUS_CUDA(cudaMemcpy(m->tables[r].ptr, ptrs.data(), m->tables[r].bytes, cudaMemcpyHostToDevice));
    }
  }
  make_streams_events(*m);
  m->xbuf.resize(g);
  m->pbuf.resize(g);
  for (int64_t r = 0; r < g; ++r) {
    use_device(m->devices[r]);
    const int64_t ns = sharding == NUS_SHARD_SAMPLES ? m->hi[r] - m->lo[r] : n;
    m->xbuf[r].alloc(ns * sizeof(double));
    m->pbuf[r].alloc(cfg_in.n_centers * sizeof(double));
  }
  use_device(m->devices[0]);
  m->gather.alloc(static_cast<size_t>(g) * cfg_in.n_centers * sizeof(double));
  m->pfinal.alloc(cfg_in.n_centers * sizeof(double));
  NUS_CUDA(cudaDeviceSynchronize());
  return m;
}

void multi_estimate(MultiEstimator& m, const double* x, double* power) {
  const int64_t g = static_cast<int64_t>(m.parts.size()), n = m.cfg.n, K = m.cfg.k_tapers, nc = m.cfg.n_centers;
  if (m.sharding == NUS_SHARD_CHANNELS) {  // independent: one host thread per part
    std::vector<std::thread> th;
    std::vector<std::string> errs(g);
    std::vector<int> codes(g, 0);
    for (int64_t r = 0; r < g; ++r)
      th.emplace_back([&, r] {
        try {
          estimator_estimate_host(*m.parts[r], x + m.lo[r] * n, power + m.lo[r] * nc, nullptr);
        } catch (const Failure& f) {
          codes[r] = f.code;
          errs[r] = f.what();
        }
      });
    for (auto& t : th) t.join();
    for (int64_t r = 0; r < g; ++r)
      if (codes[r]) fail(codes[r], errs[r]);
    return;
  }
  if (m.sharding == NUS_SHARD_TAPERS) {
    for (int64_t r = 0; r < g; ++r) {
      Estimator& e = *m.parts[r];
      use_device(m.devices[r]);
      cudaStream_t s = m.streams[r];
      NUS_CUDA(cudaMemcpyAsync(m.xbuf[r].ptr, x, n * sizeof(double), cudaMemcpyHostToDevice, s));
      const int64_t kg = m.hi[r] - m.lo[r];
      SpreadArgs a;
      a.x = m.xbuf[r].ptr;
      a.tapers = e.tapers_sorted.ptr;
      a.k = kg;
      a.kpad = kg;
      a.grid = e.grid.ptr;
      launch_spread(*e.plan, a, s);
      run_transform(*e.plan, e.grid.ptr, kg, kg, nullptr, m.pbuf[r].ptr, true, static_cast<double>(K), false, s);
      NUS_CUDA(cudaEventRecord(m.ev_pdone[r], s));
    }
    reduce_partials(m, power);
    return;
  }
  // ---- samples: fused spread -> peer slots, slot sums, owned transforms, partial-P reduce
  const int b = m.parity;
  m.parity ^= 1;
  for (int64_t r = 0; r < g; ++r) {
    Estimator& e = *m.parts[r];
    use_device(m.devices[r]);
    cudaStream_t s = m.streams[r];
    const int64_t ns = m.hi[r] - m.lo[r];
    NUS_CUDA(cudaMemcpyAsync(m.xbuf[r].ptr, x + m.lo[r], ns * sizeof(double), cudaMemcpyHostToDevice, s));
    if (m.used[b])  // parity b's slots were last read by every owner's sum two spectra ago
      for (int64_t o = 0; o < g; ++o) NUS_CUDA(cudaStreamWaitEvent(s, m.ev_sum[b][o], 0));
    SpreadArgs a;
    a.x = m.xbuf[r].ptr;
    a.tapers = e.tapers_sorted.ptr;
    a.k = K;
    a.kpad = K;
    a.grid = nullptr;
    a.slots = static_cast<void* const*>(m.tables[r].ptr) + b * g;
    a.per = m.per;
    launch_spread(*e.plan, a, s);
    NUS_CUDA(cudaEventRecord(m.ev_spread[r], s));
  }
  m.used[b] = true;
  const Plan& p0 = *m.parts[0]->plan;
  const size_t cb = p0.p.precision == NUS_F64 ? sizeof(double2) : sizeof(float2);
  const int64_t count = m.per * p0.p.mr;
  for (int64_t o = 0; o < g; ++o) {
    Estimator& e = *m.parts[o];
    use_device(m.devices[o]);
    cudaStream_t s = m.streams[o];
    for (int64_t r = 0; r < g; ++r) NUS_CUDA(cudaStreamWaitEvent(s, m.ev_spread[r], 0));
    sum_slots(static_cast<char*>(m.recv[o].ptr) + b * g * count * cb, g, count, count, m.owned[o].ptr,
              p0.p.precision == NUS_F64, s);
    NUS_CUDA(cudaEventRecord(m.ev_sum[b][o], s));
    const int64_t k0 = o * m.per, k1 = std::min(K, k0 + m.per);
    if (k1 > k0)
      run_transform(*e.plan, m.owned[o].ptr, k1 - k0, k1 - k0, nullptr, m.pbuf[o].ptr, true, static_cast<double>(K),
                    false, s);
    else
      NUS_CUDA(cudaMemsetAsync(m.pbuf[o].ptr, 0, nc * sizeof(double), s));
    NUS_CUDA(cudaEventRecord(m.ev_pdone[o], s));
  }
  reduce_partials(m, power);
}

int64_t multi_peer_bytes(const MultiEstimator& m) {
  if (m.sharding == NUS_SHARD_CHANNELS) return 0;
  const int64_t g = static_cast<int64_t>(m.parts.size()), nc = m.cfg.n_centers, K = m.cfg.k_tapers;
  if (m.sharding == NUS_SHARD_TAPERS) return (g - 1) * nc * 8;
  const Plan& p0 = *m.parts[0]->plan;
  const int64_t cb = p0.p.precision == NUS_F64 ? 16 : 8;
  // part r stores the occupied rows of every taper it does not own into that owner's slot
  const int64_t cells = p0.ffft.blocked ? static_cast<int64_t>(p0.ffft.row_cnt) * (p0.p.mr / p0.ffft.R) : p0.p.mr;
  int64_t foreign = 0;
  for (int64_t r = 0; r < g; ++r) {
    const int64_t k0 = r * m.per, k1 = std::min(K, k0 + m.per);
    foreign += K - std::max<int64_t>(0, k1 - k0);
  }
  return foreign * cells * cb + (g - 1) * nc * 8;
}

void multi_tapers(const MultiEstimator& m, double* out) {
  std::memcpy(out, m.tapers.data(), m.tapers.size() * sizeof(double));
}

}  // namespace nus
