// Multi-GPU batch registration (include/dreg_cuda.h).
//
// Pairs are independent, so the box's devices split a batch into contiguous shards,
// one host thread per device driving that device's own context (engine.cu); no field
// data ever crosses devices.  Each device writes a fixed-size dreg_pair_record per
// pair from its pair state on the device; ONE ncclAllGather over the communicator
// clique (ncclCommInitAll: NVLink / NVSwitch inside the box) then gives every device
// all records, and device 0's copy is returned to the caller in pair order.
//
// NCCL is resolved with dlopen("libnccl.so.2") at dreg_cuda_multi_create, so the
// single-device library has no link-time NCCL dependency (and a process that
// already loaded torch's NCCL reuses that copy).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "dreg_cuda.h"
#include "engine_internal.h"

namespace {

struct Nccl {
    void* so = nullptr;
    decltype(&ncclCommInitAll) comm_init_all = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;

    bool load(std::string& err) {
        if (so) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (so) break;
        }
        if (!so) {
            err = std::string("NCCL not found (dlopen libnccl.so.2): ") + dlerror();
            return false;
        }
        comm_init_all = reinterpret_cast<decltype(comm_init_all)>(dlsym(so, "ncclCommInitAll"));
        comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(so, "ncclCommDestroy"));
        all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(so, "ncclAllGather"));
        group_start = reinterpret_cast<decltype(group_start)>(dlsym(so, "ncclGroupStart"));
        group_end = reinterpret_cast<decltype(group_end)>(dlsym(so, "ncclGroupEnd"));
        error_string = reinterpret_cast<decltype(error_string)>(dlsym(so, "ncclGetErrorString"));
        if (!comm_init_all || !comm_destroy || !all_gather || !group_start || !group_end || !error_string) {
            err = "libnccl.so.2 lacks ncclCommInitAll / ncclAllGather / ncclGroupStart";
            return false;
        }
        return true;
    }
};

Nccl& nccl() {
    static Nccl n;
    return n;
}

dreg_pair_record padding_record() {
    dreg_pair_record r;
    std::memset(&r, 0, sizeof r);
    r.pair = -1;
    r.device = -1;
    return r;
}

}  // namespace

struct dreg_cuda_multi {
    std::vector<int> devices;
    std::vector<dreg_cuda_ctx*> ctx;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
    std::vector<dreg_pair_record*> send, recv;  // device buffers: cap / n * cap records
    int cap = 0;
    std::string err;

    void free_buffers() {
        for (size_t d = 0; d < devices.size(); ++d) {
            cudaSetDevice(devices[d]);
            if (d < send.size() && send[d]) cudaFree(send[d]);
            if (d < recv.size() && recv[d]) cudaFree(recv[d]);
        }
        send.assign(devices.size(), nullptr);
        recv.assign(devices.size(), nullptr);
        cap = 0;
    }
};

namespace {

int fail(dreg_cuda_multi* m, int code, const std::string& msg) {
    if (m) m->err = msg;
    return code;
}

bool cuda_ok(dreg_cuda_multi* m, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return true;
    m->err = std::string(what) + ": " + cudaGetErrorString(e);
    return false;
}

}  // namespace

extern "C" {

int dreg_shard_range(int n_pairs, int n_shards, int shard, int* begin, int* end) {
    if (n_pairs < 0 || n_shards < 1 || shard < 0 || shard >= n_shards || !begin || !end)
        return DREG_INVALID_ARGUMENT;
    *begin = (int)(((long long)shard * n_pairs) / n_shards);
    *end = (int)(((long long)(shard + 1) * n_pairs) / n_shards);
    return DREG_OK;
}

int dreg_records_unpack(const dreg_pair_record* gathered, int n_shards, int cap, int n_pairs,
                        dreg_pair_record* out) {
    if (n_shards < 1 || cap < 0 || n_pairs < 0 || (n_pairs > 0 && (!gathered || !out)))
        return DREG_INVALID_ARGUMENT;
    std::vector<char> seen((size_t)n_pairs, 0);
    for (int s = 0; s < n_shards; ++s) {
        int b = 0, e = 0;
        dreg_shard_range(n_pairs, n_shards, s, &b, &e);
        if (e - b > cap) return DREG_INVALID_ARGUMENT;
        for (int i = 0; i < cap; ++i) {
            const dreg_pair_record& r = gathered[(size_t)s * cap + i];
            if (i >= e - b) {
                if (r.pair != -1) return DREG_INVALID_ARGUMENT;  // padding must stay padding
                continue;
            }
            if (r.pair != b + i || seen[(size_t)r.pair]) return DREG_INVALID_ARGUMENT;
            seen[(size_t)r.pair] = 1;
            out[r.pair] = r;
        }
    }
    for (char v : seen)
        if (!v) return DREG_INVALID_ARGUMENT;
    return DREG_OK;
}

int dreg_cuda_multi_create(const int* devices, int n_devices, dreg_cuda_multi** out) {
    if (!out || !devices || n_devices < 1) return DREG_INVALID_ARGUMENT;
    *out = nullptr;
    int have = 0;
    if (cudaGetDeviceCount(&have) != cudaSuccess || have <= 0) return DREG_RUNTIME;
    for (int i = 0; i < n_devices; ++i) {
        if (devices[i] < 0 || devices[i] >= have) return DREG_INVALID_ARGUMENT;
        for (int j = 0; j < i; ++j)
            if (devices[j] == devices[i]) return DREG_INVALID_ARGUMENT;  // one rank per device
    }
    auto* m = new dreg_cuda_multi();
    m->devices.assign(devices, devices + n_devices);
    m->ctx.assign(n_devices, nullptr);
    m->send.assign(n_devices, nullptr);
    m->recv.assign(n_devices, nullptr);
    auto bail = [&](int code) {
        dreg_cuda_multi_destroy(m);
        return code;
    };
    for (int d = 0; d < n_devices; ++d) {
        const int st = dreg_cuda_ctx_create(devices[d], &m->ctx[d]);
        if (st != DREG_OK) return bail(st);
    }
    std::string err;
    if (!nccl().load(err)) return bail(DREG_RUNTIME);
    m->comms.assign(n_devices, nullptr);
    if (nccl().comm_init_all(m->comms.data(), n_devices, devices) != ncclSuccess) {
        m->comms.clear();
        return bail(DREG_RUNTIME);
    }
    m->streams.assign(n_devices, nullptr);
    for (int d = 0; d < n_devices; ++d) {
        if (cudaSetDevice(devices[d]) != cudaSuccess ||
            cudaStreamCreateWithFlags(&m->streams[d], cudaStreamNonBlocking) != cudaSuccess)
            return bail(DREG_RUNTIME);
    }
    *out = m;
    return DREG_OK;
}

void dreg_cuda_multi_destroy(dreg_cuda_multi* m) {
    if (!m) return;
    m->free_buffers();
    for (size_t d = 0; d < m->comms.size(); ++d)
        if (m->comms[d]) nccl().comm_destroy(m->comms[d]);
    for (size_t d = 0; d < m->streams.size(); ++d)
        if (m->streams[d]) {
            cudaSetDevice(m->devices[d]);
            cudaStreamDestroy(m->streams[d]);
        }
    for (dreg_cuda_ctx* c : m->ctx)
        if (c) dreg_cuda_ctx_destroy(c);
    delete m;
}

const char* dreg_cuda_multi_last_error(const dreg_cuda_multi* m) { return m ? m->err.c_str() : "null handle"; }

int dreg_cuda_multi_device_count(const dreg_cuda_multi* m) { return m ? (int)m->devices.size() : 0; }

int dreg_cuda_multi_register_batch(dreg_cuda_multi* m, int n_pairs, const float* const* targets,
                                   const float* const* sources, dreg_dims3 dims, dreg_spacing3 spacing,
                                   const dreg_reg_cfg* cfg, float* const* phi_out, float* const* warped_out,
                                   dreg_pair_result* results, dreg_pair_record* records) {
    if (!m) return DREG_INVALID_ARGUMENT;
    if (!(spacing.x > 0.0) || !(spacing.y > 0.0) || !(spacing.z > 0.0))
        return fail(m, DREG_INVALID_ARGUMENT, "voxel spacing must be positive");
    if (n_pairs < 0) return fail(m, DREG_INVALID_ARGUMENT, "n_pairs must be >= 0");
    if (n_pairs > 0 && (!targets || !sources)) return fail(m, DREG_INVALID_ARGUMENT, "null input arrays");
    const int D = (int)m->devices.size();
    std::vector<int> b(D), e(D);
    int cap = 0;
    for (int d = 0; d < D; ++d) {
        dreg_shard_range(n_pairs, D, d, &b[d], &e[d]);
        cap = std::max(cap, e[d] - b[d]);
    }
    cap = std::max(cap, 1);
    if (cap > m->cap) {  // gather buffers: send [cap], recv [D][cap] per device
        m->free_buffers();
        for (int d = 0; d < D; ++d) {
            if (!cuda_ok(m, cudaSetDevice(m->devices[d]), "cudaSetDevice") ||
                !cuda_ok(m, cudaMalloc(&m->send[d], sizeof(dreg_pair_record) * cap), "cudaMalloc") ||
                !cuda_ok(m, cudaMalloc(&m->recv[d], sizeof(dreg_pair_record) * cap * D), "cudaMalloc"))
                return DREG_RUNTIME;
        }
        m->cap = cap;
    }
    cap = m->cap;
    // one host thread per device: its shard through its own context
    std::vector<int> status(D, DREG_OK);
    std::vector<std::string> errs(D);
    const std::vector<dreg_pair_record> pad((size_t)cap, padding_record());
    auto work = [&](int d) {
        try {
            if (cudaSetDevice(m->devices[d]) != cudaSuccess ||
                cudaMemcpy(m->send[d], pad.data(), sizeof(dreg_pair_record) * cap, cudaMemcpyHostToDevice) !=
                    cudaSuccess) {
                status[d] = DREG_RUNTIME;
                errs[d] = "device setup failed";
                return;
            }
            const int n = e[d] - b[d];
            status[d] = dregb_register_batch_records(
                m->ctx[d], n, n ? targets + b[d] : nullptr, n ? sources + b[d] : nullptr, dims, cfg,
                phi_out ? phi_out + b[d] : nullptr, warped_out ? warped_out + b[d] : nullptr,
                results ? results + b[d] : nullptr, m->send[d], b[d], m->devices[d]);
            if (status[d] != DREG_OK) errs[d] = dreg_cuda_last_error(m->ctx[d]);
        } catch (const std::exception& ex) {
            status[d] = DREG_RUNTIME;
            errs[d] = ex.what();
        }
    };
    std::vector<std::thread> threads;
    for (int d = 1; d < D; ++d) threads.emplace_back(work, d);
    work(0);
    for (auto& t : threads) t.join();
    int first_bad = DREG_OK;
    for (int d = 0; d < D; ++d) {
        if (status[d] == DREG_OK || status[d] == DREG_NUMERIC) {
            if (status[d] == DREG_NUMERIC && first_bad == DREG_OK) {
                first_bad = DREG_NUMERIC;
                m->err = "device " + std::to_string(m->devices[d]) + ": " + errs[d];
            }
            continue;
        }
        return fail(m, status[d], "device " + std::to_string(m->devices[d]) + ": " + errs[d]);
    }
    // the one collective: all-gather of the per-pair records (grouped: one thread, D comms)
    if (nccl().group_start() != ncclSuccess) return fail(m, DREG_RUNTIME, "ncclGroupStart failed");
    for (int d = 0; d < D; ++d) {
        cudaSetDevice(m->devices[d]);
        const ncclResult_t r = nccl().all_gather(m->send[d], m->recv[d], sizeof(dreg_pair_record) * cap, ncclUint8,
                                                 m->comms[d], m->streams[d]);
        if (r != ncclSuccess) {
            nccl().group_end();
            return fail(m, DREG_RUNTIME, std::string("ncclAllGather: ") + nccl().error_string(r));
        }
    }
    if (nccl().group_end() != ncclSuccess) return fail(m, DREG_RUNTIME, "ncclGroupEnd failed");
    for (int d = 0; d < D; ++d) {
        if (!cuda_ok(m, cudaSetDevice(m->devices[d]), "cudaSetDevice") ||
            !cuda_ok(m, cudaStreamSynchronize(m->streams[d]), "all-gather"))
            return DREG_RUNTIME;
    }
    if (records && n_pairs > 0) {
        std::vector<dreg_pair_record> all((size_t)D * cap);
        cudaSetDevice(m->devices[0]);
        if (!cuda_ok(m, cudaMemcpy(all.data(), m->recv[0], sizeof(dreg_pair_record) * all.size(),
                                   cudaMemcpyDeviceToHost),
                     "gathered records"))
            return DREG_RUNTIME;
        if (dreg_records_unpack(all.data(), D, cap, n_pairs, records) != DREG_OK)
            return fail(m, DREG_RUNTIME, "all-gather returned an inconsistent record layout");
    }
    if (first_bad == DREG_OK) m->err.clear();
    return first_bad;
}

}  // extern "C"
