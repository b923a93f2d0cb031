// gd_multi.cpp -- query-row sharding over several B200s.
//
// Under full_deadline every app's selection depends on that app alone
// (scheduler.cpp:203-205: the budget is the job's own deadline), so the grid
// path shards by contiguous app ranges with a replica of both packed
// ensembles per device and needs exactly ONE collective: a gather of the
// 24-byte per-app decisions to the root device.  Two forms:
//
//   gd_comm   one process per GPU (torchrun): ncclCommInitRank over a shared
//             unique id; gd_gather_decisions enqueues the gather on the
//             context stream.
//   gd_multi  one process driving N GPUs: a context per device,
//             ncclCommInitAll, one host thread per device running the
//             host-buffer grid call on its range, then the gather and one
//             device-to-host copy from the root.
//
// NCCL is loaded at first use (dlopen): the library itself keeps no link-time
// NCCL dependency, and a process that already loaded NCCL (torch) shares that
// copy.  ncclGather (NCCL >= 2.28) is used when every rank sends the same
// count; otherwise -- or with an older NCCL -- the gather is the grouped
// ncclSend / ncclRecv form (same single collective step).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gd_host.hpp"

namespace {

typedef int nccl_result;
typedef struct nccl_comm_opaque* nccl_comm;
struct nccl_uid {
    char internal[128];
};
constexpr int kNcclInt8 = 0;

struct Nccl {
    bool ok = false;
    std::string why;
    nccl_result (*get_unique_id)(nccl_uid*) = nullptr;
    nccl_result (*init_rank)(nccl_comm*, int, nccl_uid, int) = nullptr;
    nccl_result (*init_all)(nccl_comm*, int, const int*) = nullptr;
    nccl_result (*destroy)(nccl_comm) = nullptr;
    nccl_result (*group_start)() = nullptr;
    nccl_result (*group_end)() = nullptr;
    nccl_result (*send)(const void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*recv)(void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*gather)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;  // >= 2.28
    const char* (*error_string)(nccl_result) = nullptr;
    nccl_result (*get_version)(int*) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        if (const char* p = std::getenv("GDVFS_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already loaded (e.g. by torch)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
        n.init_rank = reinterpret_cast<decltype(n.init_rank)>(sym("ncclCommInitRank"));
        n.init_all = reinterpret_cast<decltype(n.init_all)>(sym("ncclCommInitAll"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("ncclCommDestroy"));
        n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
        n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
        n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
        n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
        n.gather = reinterpret_cast<decltype(n.gather)>(sym("ncclGather"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
        n.get_version = reinterpret_cast<decltype(n.get_version)>(sym("ncclGetVersion"));
        n.ok = n.get_unique_id && n.init_rank && n.init_all && n.destroy && n.group_start && n.group_end && n.send &&
               n.recv && n.error_string;
        if (!n.ok) n.why = "libnccl.so.2 lacks a required symbol";
    });
    return n;
}

int nccl_error(nccl_result r, const char* where) {
    const Nccl& n = nccl();
    return gdh::set_error(GD_ERR_CUDA, std::string(where) + ": " + (n.error_string ? n.error_string(r) : "nccl error"));
}

int need_nccl() {
    const Nccl& n = nccl();
    return n.ok ? GD_OK : gdh::set_error(GD_ERR_UNSUPPORTED, "NCCL unavailable: " + n.why);
}

// Rank g of G owns apps [a0, a1): contiguous, sizes differ by at most one
// (paper_2004_08177_b200/shard.py shard_range, the same split).
void shard_range(int64_t n, int g, int G, int64_t& a0, int64_t& a1) {
    a0 = n * g / G;
    a1 = n * (g + 1) / G;
}

// The one collective: rank r's count[r] decisions land at recv + off[r] on
// `root`.  `per_rank` lists (comm, stream, send, recv) of every rank this
// process drives (one entry for gd_comm, N for gd_multi).
struct RankIo {
    nccl_comm comm;
    cudaStream_t stream;
    int rank;
    const gd_decision* send;
    gd_decision* recv;  // root only
};

int gather(const std::vector<RankIo>& io, int n_ranks, int root, const std::vector<int64_t>& counts) {
    const Nccl& n = nccl();
    bool equal = true;
    for (int64_t c : counts) equal = equal && c == counts[0];
    nccl_result r = n.group_start();
    if (r) return nccl_error(r, "ncclGroupStart");
    for (const RankIo& x : io) {
        if (equal && n.gather) {
            r = n.gather(x.send, x.recv, static_cast<size_t>(counts[0]) * sizeof(gd_decision), kNcclInt8, root, x.comm,
                         x.stream);
            if (r) break;
            continue;
        }
        if (x.rank == root) {
            int64_t off = 0;
            for (int q = 0; q < n_ranks && !r; ++q) {
                const size_t bytes = static_cast<size_t>(counts[static_cast<size_t>(q)]) * sizeof(gd_decision);
                if (q == root) {
                    if (bytes) {
                        cudaError_t e = cudaMemcpyAsync(x.recv + off, x.send, bytes, cudaMemcpyDeviceToDevice, x.stream);
                        if (e != cudaSuccess) {
                            n.group_end();
                            return gdh::cuda_error(e, "gather (root copy)");
                        }
                    }
                } else if (bytes) {
                    r = n.recv(x.recv + off, bytes, kNcclInt8, q, x.comm, x.stream);
                }
                off += counts[static_cast<size_t>(q)];
            }
        } else {
            const size_t bytes = static_cast<size_t>(counts[static_cast<size_t>(x.rank)]) * sizeof(gd_decision);
            if (bytes) r = n.send(x.send, bytes, kNcclInt8, root, x.comm, x.stream);
        }
        if (r) break;
    }
    const nccl_result r2 = n.group_end();
    if (r) return nccl_error(r, "gather");
    if (r2) return nccl_error(r2, "ncclGroupEnd");
    return GD_OK;
}

}  // namespace

struct gd_comm {
    gd_ctx* ctx = nullptr;  // not owned
    nccl_comm comm = nullptr;
    int32_t n_ranks = 0, rank = 0;
};

struct gd_multi {
    std::vector<gd_ctx*> ctxs;  // owned, one per device
    std::vector<nccl_comm> comms;
};

extern "C" {

int gd_comm_unique_id(void* id128) {
    if (!id128) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_comm_unique_id: null out");
    int rc = need_nccl();
    if (rc) return rc;
    nccl_uid uid;
    nccl_result r = nccl().get_unique_id(&uid);
    if (r) return nccl_error(r, "ncclGetUniqueId");
    std::memcpy(id128, uid.internal, sizeof(uid.internal));
    return GD_OK;
}

int gd_comm_init_rank(gd_ctx* ctx, const void* id128, int32_t n_ranks, int32_t rank, gd_comm** out) {
    if (!ctx || !id128 || !out || n_ranks < 1 || rank < 0 || rank >= n_ranks) {
        return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_comm_init_rank: bad argument");
    }
    *out = nullptr;
    int rc = need_nccl();
    if (rc) return rc;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return gdh::cuda_error(e, "cudaSetDevice");
    nccl_uid uid;
    std::memcpy(uid.internal, id128, sizeof(uid.internal));
    auto* c = new gd_comm;
    c->ctx = ctx;
    c->n_ranks = n_ranks;
    c->rank = rank;
    nccl_result r = nccl().init_rank(&c->comm, n_ranks, uid, rank);
    if (r) {
        delete c;
        return nccl_error(r, "ncclCommInitRank");
    }
    *out = c;
    return GD_OK;
}

int gd_comm_destroy(gd_comm* comm) {
    if (!comm) return GD_OK;
    cudaSetDevice(comm->ctx->device);
    if (comm->comm) nccl().destroy(comm->comm);
    delete comm;
    return GD_OK;
}

int gd_gather_decisions(gd_comm* comm, const gd_decision* d_send, const int64_t* counts, gd_decision* d_recv,
                        int32_t root) {
    if (!comm || !counts || root < 0 || root >= comm->n_ranks) {
        return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_gather_decisions: bad argument");
    }
    std::vector<int64_t> cnt(counts, counts + comm->n_ranks);
    for (int64_t c : cnt) {
        if (c < 0) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_gather_decisions: negative count");
    }
    if ((cnt[static_cast<size_t>(comm->rank)] > 0 && !d_send) || (comm->rank == root && !d_recv)) {
        return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_gather_decisions: null buffer");
    }
    cudaError_t e = cudaSetDevice(comm->ctx->device);
    if (e != cudaSuccess) return gdh::cuda_error(e, "cudaSetDevice");
    if (comm->n_ranks == 1) {  // no peers: the gather is a local copy
        if (cnt[0] > 0 && d_recv != d_send) {
            e = cudaMemcpyAsync(d_recv, d_send, static_cast<size_t>(cnt[0]) * sizeof(gd_decision),
                                cudaMemcpyDeviceToDevice, comm->ctx->stream);
            if (e != cudaSuccess) return gdh::cuda_error(e, "gather (local copy)");
        }
        return GD_OK;
    }
    int rc = need_nccl();
    if (rc) return rc;
    return gather({RankIo{comm->comm, comm->ctx->stream, comm->rank, d_send, d_recv}}, comm->n_ranks, root, cnt);
}

int gd_multi_create(const int32_t* devices, int32_t n_devices, gd_multi** out) {
    if (!devices || n_devices < 1 || !out) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_multi_create: bad argument");
    *out = nullptr;
    auto* m = new gd_multi;
    for (int32_t g = 0; g < n_devices; ++g) {
        for (int32_t h = 0; h < g; ++h) {
            if (devices[h] == devices[g]) {
                gd_multi_destroy(m);
                return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_multi_create: duplicate device");
            }
        }
        gd_ctx* c = nullptr;
        int rc = gd_ctx_create(devices[g], &c);
        if (rc) {
            gd_multi_destroy(m);
            return rc;
        }
        m->ctxs.push_back(c);
    }
    if (n_devices > 1) {
        int rc = need_nccl();
        if (rc) {
            gd_multi_destroy(m);
            return rc;
        }
        m->comms.assign(static_cast<size_t>(n_devices), nullptr);
        nccl_result r = nccl().init_all(m->comms.data(), n_devices, devices);
        if (r) {
            m->comms.clear();
            gd_multi_destroy(m);
            return nccl_error(r, "ncclCommInitAll");
        }
    }
    *out = m;
    return GD_OK;
}

int gd_multi_destroy(gd_multi* m) {
    if (!m) return GD_OK;
    for (size_t g = 0; g < m->comms.size(); ++g) {
        if (m->comms[g]) {
            cudaSetDevice(m->ctxs[g]->device);
            nccl().destroy(m->comms[g]);
        }
    }
    for (gd_ctx* c : m->ctxs) gd_ctx_destroy(c);
    delete m;
    return GD_OK;
}

int32_t gd_multi_size(const gd_multi* m) { return m ? static_cast<int32_t>(m->ctxs.size()) : 0; }

int gd_multi_ctx(gd_multi* m, int32_t i, gd_ctx** out) {
    if (!m || !out || i < 0 || i >= gd_multi_size(m)) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_multi_ctx: bad index");
    *out = m->ctxs[static_cast<size_t>(i)];
    return GD_OK;
}

int gd_multi_model_replicate(gd_multi* m, const gd_model* src, gd_model** replicas) {
    if (!m || !src || !replicas) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_multi_model_replicate: null argument");
    const size_t G = m->ctxs.size();
    for (size_t g = 0; g < G; ++g) replicas[g] = nullptr;
    for (size_t g = 0; g < G; ++g) {
        int rc = gdh::clone_model(m->ctxs[g], src, &replicas[g]);
        if (rc) {
            for (size_t h = 0; h < g; ++h) {
                gd_model_free(replicas[h]);
                replicas[h] = nullptr;
            }
            return rc;
        }
    }
    return GD_OK;
}

int gd_multi_grid_select(gd_multi* m, gd_model* const* energy, gd_model* const* time, const gd_grid* g,
                         const gd_select_opts* o, gd_decision* out, double* e_out, double* t_out) {
    if (!m || !energy || !time || !g || !o) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "gd_multi_grid_select: null argument");
    const int G = static_cast<int>(m->ctxs.size());
    const int64_t A = g->n_apps, C = g->n_clocks;
    if (A < 0) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: negative sizes");
    if (A > 0 && !out) return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: null decisions");
    if (!g->rec_of_clock && g->n_records < A) {
        return gdh::set_error(GD_ERR_INVALID_ARGUMENT, "grid_select: one record per app required without rec_of_clock");
    }
    // Per-device sub-grids: without rec_of_clock record a is app a, so a
    // shard ships only its own rows; with it, every record stays addressable.
    std::vector<gd_grid> sub(static_cast<size_t>(G), *g);
    std::vector<int64_t> counts(static_cast<size_t>(G));
    std::vector<int64_t> first(static_cast<size_t>(G));
    for (int r = 0; r < G; ++r) {
        int64_t a0, a1;
        shard_range(A, r, G, a0, a1);
        gd_grid& s = sub[static_cast<size_t>(r)];
        s.n_apps = a1 - a0;
        s.budgets = g->budgets ? g->budgets + a0 : nullptr;
        if (g->rec_of_clock) {
            s.rec_of_clock = g->rec_of_clock + a0 * C;
        } else {
            s.rows = g->rows ? g->rows + a0 * g->n_cols : nullptr;
            s.cat_t = g->cat_t ? g->cat_t + a0 * g->n_cat : nullptr;
            s.n_records = a1 - a0;
        }
        counts[static_cast<size_t>(r)] = a1 - a0;
        first[static_cast<size_t>(r)] = a0;
    }
    // One host thread per device: host-buffer call on its range (H2D of its
    // rows, kernels, optional E/T tables straight into the caller's arrays),
    // decisions left on the device for the gather.
    std::vector<int> rcs(static_cast<size_t>(G), GD_OK);
    std::vector<std::string> errs(static_cast<size_t>(G));
    std::vector<gd_decision*> dev_out(static_cast<size_t>(G), nullptr);
    auto work = [&](int r) {
        const size_t i = static_cast<size_t>(r);
        const int64_t a0 = first[i];
        rcs[i] = gdh::grid_select_host(m->ctxs[i], energy[i], time[i], &sub[i], o, nullptr,
                                       e_out ? e_out + a0 * C : nullptr, t_out ? t_out + a0 * C : nullptr, &dev_out[i]);
        if (rcs[i]) errs[i] = gd_last_error();
    };
    if (G == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int r = 0; r < G; ++r) th.emplace_back(work, r);
        for (auto& t : th) t.join();
    }
    for (int r = 0; r < G; ++r) {
        if (rcs[static_cast<size_t>(r)]) {
            return gdh::set_error(rcs[static_cast<size_t>(r)],
                                  "device " + std::to_string(m->ctxs[static_cast<size_t>(r)]->device) + ": " +
                                      errs[static_cast<size_t>(r)]);
        }
    }
    if (A == 0) return GD_OK;
    gd_ctx* root = m->ctxs[0];
    const size_t bytes = static_cast<size_t>(A) * sizeof(gd_decision);
    // Root receive buffer (stream-ordered), then one copy to the caller.
    cudaError_t e = cudaSetDevice(root->device);
    if (e != cudaSuccess) return gdh::cuda_error(e, "cudaSetDevice");
    gd_decision* recv = nullptr;
    if (G == 1) {
        recv = dev_out[0];
    } else {
        e = cudaMallocAsync(reinterpret_cast<void**>(&recv), bytes, root->stream);
        if (e != cudaSuccess) return gdh::cuda_error(e, "cudaMallocAsync(gather)");
        std::vector<RankIo> io;
        for (int r = 0; r < G; ++r) {
            const size_t i = static_cast<size_t>(r);
            io.push_back(RankIo{m->comms[i], m->ctxs[i]->stream, r, dev_out[i], r == 0 ? recv : nullptr});
        }
        int rc = gather(io, G, 0, counts);
        if (rc) {
            cudaFreeAsync(recv, root->stream);
            return rc;
        }
    }
    e = cudaMemcpyAsync(out, recv, bytes, cudaMemcpyDeviceToHost, root->stream);
    if (G > 1) cudaFreeAsync(recv, root->stream);
    if (e != cudaSuccess) return gdh::cuda_error(e, "D2H decisions");
    for (int r = 0; r < G; ++r) {
        cudaSetDevice(m->ctxs[static_cast<size_t>(r)]->device);
        e = cudaStreamSynchronize(m->ctxs[static_cast<size_t>(r)]->stream);
        if (e != cudaSuccess) return gdh::cuda_error(e, "multi sync");
    }
    return GD_OK;
}

}  // extern "C"
