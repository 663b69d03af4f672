// bltc_run_distributed: decomp.run_distributed (decomp.py:483-593) behind the
// C ABI, for hosts that do not run one process per GPU: R ranks on the given
// devices in one process (rank r on devices[r % n_devices]), one host thread
// per rank.  Each rank builds its tree / batches / moments from its RCB slice
// (the caller's order: rcb_order[rank_start[r] .. rank_start[r+1]), e.g. the
// reference's rcb_partition), publishes its records / particles / moment rows
// on its own device, and evaluates its batches against every rank's published
// buffers -- read across devices by the copies in bltc_rank_evaluate (peer
// access over NVLink when enabled, staged otherwise) -- in the reference's
// owner order.  phi comes back in the original particle order.
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "bltc_internal.cuh"

namespace {

struct RankBufs {
  bltc_ctx* ctx = nullptr;
  int device = 0;
  int64_t n = 0;
  bltc_publish_sizes sz{};
  double* records = nullptr;
  double* particles = nullptr;
  double* moments = nullptr;
  std::vector<double> x, y, z, q, phi;
  bltc_stats st{};
  int rc = BLTC_OK;
  std::string err;
};

template <typename F>
void run_ranks(std::vector<RankBufs>& R, F&& f) {
  std::vector<std::thread> th;
  for (size_t r = 0; r < R.size(); ++r)
    th.emplace_back([&, r] {
      if (R[r].rc == BLTC_OK) {
        R[r].rc = f(R[r], (int)r);
        if (R[r].rc != BLTC_OK) R[r].err = bltc_last_error();
      }
    });
  for (auto& t : th) t.join();
}

int first_error(const std::vector<RankBufs>& R) {
  for (const auto& b : R)
    if (b.rc != BLTC_OK) {
      bltc::set_error(b.err);
      return b.rc;
    }
  return BLTC_OK;
}

}  // namespace

extern "C" BLTC_API int bltc_run_distributed(int32_t ranks, const int32_t* devices,
                                             int32_t n_devices, const bltc_params* p,
                                             const double* cheb_s, int64_t n, const double* x,
                                             const double* y, const double* z, const double* q,
                                             const int64_t* rcb_order,
                                             const int64_t* rank_start, double* phi_out,
                                             bltc_stats* stats) {
  using namespace bltc;
  if (ranks < 1 || n_devices < 1 || !devices || !p || !x || !y || !z || !q || !rcb_order ||
      !rank_start || !phi_out) {
    set_error("bltc_run_distributed: invalid arguments");
    return BLTC_ERR_VALUE;
  }
  if (rank_start[0] != 0 || rank_start[ranks] != n) {
    set_error("rank_start must run from 0 to n");
    return BLTC_ERR_VALUE;
  }
  for (int r = 0; r < ranks; ++r)
    if (rank_start[r + 1] - rank_start[r] < 1) {
      set_error("every rank needs at least one particle");
      return BLTC_ERR_VALUE;
    }
  for (int64_t i = 0; i < n; ++i)
    if (rcb_order[i] < 0 || rcb_order[i] >= n) {
      set_error("rcb_order out of range");
      return BLTC_ERR_VALUE;
    }
  std::vector<RankBufs> R(ranks);
  for (int r = 0; r < ranks; ++r) {
    RankBufs& b = R[r];
    b.device = devices[r % n_devices];
    b.n = rank_start[r + 1] - rank_start[r];
    b.x.resize(b.n);
    b.y.resize(b.n);
    b.z.resize(b.n);
    b.q.resize(b.n);
    b.phi.resize(b.n);
    for (int64_t k = 0; k < b.n; ++k) {
      const int64_t i = rcb_order[rank_start[r] + k];
      b.x[k] = x[i];
      b.y[k] = y[i];
      b.z[k] = z[i];
      b.q[k] = q[i];
    }
  }
  // peer access between the devices in use (NVLink); ignore "already enabled"
  for (int a = 0; a < n_devices; ++a)
    for (int c = 0; c < n_devices; ++c) {
      if (devices[a] == devices[c]) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, devices[a], devices[c]) == cudaSuccess && can) {
        cudaSetDevice(devices[a]);
        cudaDeviceEnablePeerAccess(devices[c], 0);
        cudaGetLastError();
      }
    }
  const int mstride = (((p->degree + 1) * (p->degree + 1) * (p->degree + 1) + 1) & ~1);
  // the global target set as the minimal boxes of its occupied cells on a
  // 16^3 grid: each rank publishes only the moment rows some batch in them
  // could read (bltc_rank_set_domain_boxes)
  std::vector<double> dboxes(6 * 16 * 16 * 16);
  int64_t n_dboxes = 0;
  {
    const int drc = bltc_domain_cells(n, x, y, z, 16, dboxes.data(), &n_dboxes);
    if (drc != BLTC_OK) return drc;
  }
  // build + publish, one thread per rank
  run_ranks(R, [&](RankBufs& b, int) {
    int rc = bltc_create(b.device, nullptr, &b.ctx);
    if (rc != BLTC_OK) return rc;
    rc = bltc_rank_set_domain_boxes(b.ctx, n_dboxes, dboxes.data());
    if (rc != BLTC_OK) return rc;
    rc = bltc_rank_build(b.ctx, p, cheb_s, b.n, b.x.data(), b.y.data(), b.z.data(),
                         b.q.data(), 0);
    if (rc != BLTC_OK) return rc;
    rc = bltc_rank_publish_sizes(b.ctx, &b.sz);
    if (rc != BLTC_OK) return rc;
    if (cudaSetDevice(b.device) != cudaSuccess ||
        cudaMalloc(&b.records, std::max<int64_t>(1, b.sz.n_clusters * b.sz.record_doubles) *
                                   sizeof(double)) != cudaSuccess ||
        cudaMalloc(&b.particles, std::max<int64_t>(1, 4 * b.sz.n_particles) * sizeof(double)) !=
            cudaSuccess ||
        cudaMalloc(&b.moments, std::max<int64_t>(1, b.sz.n_moment_rows * mstride) *
                                   sizeof(double)) != cudaSuccess) {
      set_error("bltc_run_distributed: device allocation failed");
      return BLTC_ERR_CUDA;
    }
    return bltc_rank_publish(b.ctx, b.records, b.particles, b.moments);
  });
  int rc = first_error(R);
  if (rc == BLTC_OK) {
    std::vector<int64_t> nc(ranks), np(ranks), nr(ranks);
    std::vector<const double*> rec(ranks), par(ranks), mom(ranks);
    for (int r = 0; r < ranks; ++r) {
      nc[r] = R[r].sz.n_clusters;
      np[r] = R[r].sz.n_particles;
      nr[r] = R[r].sz.n_moment_rows;
      rec[r] = R[r].records;
      par[r] = R[r].particles;
      mom[r] = R[r].moments;
    }
    run_ranks(R, [&](RankBufs& b, int r) {
      // owners on another device without peer access: stage their published
      // buffers onto this rank's device first (cudaMemcpyPeer); with peer
      // access the kernels and copies read them in place over NVLink
      std::vector<const double*> rr = rec, pp = par, mm = mom;
      std::vector<double*> mirrors;
      int rc = BLTC_OK;
      cudaSetDevice(b.device);
      for (int o = 0; o < ranks && rc == BLTC_OK; ++o) {
        int can = 1;
        if (R[o].device != b.device &&
            (cudaDeviceCanAccessPeer(&can, b.device, R[o].device) != cudaSuccess || !can)) {
          const int64_t sz[3] = {nc[o] * R[o].sz.record_doubles, 4 * np[o], nr[o] * mstride};
          const double* srcp[3] = {rec[o], par[o], mom[o]};
          const double** dstp[3] = {&rr[o], &pp[o], &mm[o]};
          for (int k = 0; k < 3; ++k) {
            double* d = nullptr;
            if (cudaMalloc(&d, std::max<int64_t>(1, sz[k]) * sizeof(double)) != cudaSuccess ||
                cudaMemcpyPeer(d, b.device, srcp[k], R[o].device, sz[k] * sizeof(double)) !=
                    cudaSuccess) {
              set_error("bltc_run_distributed: staging a remote rank's buffers failed");
              rc = BLTC_ERR_CUDA;
            }
            if (d) mirrors.push_back(d);
            *dstp[k] = d;
          }
        }
      }
      if (rc == BLTC_OK)
        rc = bltc_rank_evaluate(b.ctx, p, ranks, r, nc.data(), np.data(), nr.data(), rr.data(),
                                pp.data(), mm.data(), b.phi.data(), 0, &b.st);
      cudaSetDevice(b.device);
      for (double* d : mirrors) cudaFree(d);
      return rc;
    });
    rc = first_error(R);
  }
  if (rc == BLTC_OK) {
    bltc_stats tot{};
    for (int r = 0; r < ranks; ++r) {
      for (int64_t k = 0; k < R[r].n; ++k) phi_out[rcb_order[rank_start[r] + k]] = R[r].phi[k];
      tot.n_clusters += R[r].st.n_clusters;
      tot.n_batches += R[r].st.n_batches;
      tot.direct_pairs += R[r].st.direct_pairs;
      tot.approx_pairs += R[r].st.approx_pairs;
      tot.n_moments += R[r].st.n_moments;
      tot.kernel_launches += R[r].st.kernel_launches;
      tot.setup_s = std::max(tot.setup_s, R[r].st.setup_s);
      tot.compute_s = std::max(tot.compute_s, R[r].st.compute_s);
      tot.total_s = std::max(tot.total_s, R[r].st.total_s);
      tot.far_s = std::max(tot.far_s, R[r].st.far_s);
      tot.near_s = std::max(tot.near_s, R[r].st.near_s);
    }
    if (stats) *stats = tot;
  }
  for (auto& b : R) {
    if (b.records || b.particles || b.moments) cudaSetDevice(b.device);
    if (b.records) cudaFree(b.records);
    if (b.particles) cudaFree(b.particles);
    if (b.moments) cudaFree(b.moments);
    if (b.ctx) bltc_destroy(b.ctx);
  }
  return rc;
}
