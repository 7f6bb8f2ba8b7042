// transport.cuh -- the communication step of one ADMM iteration between ranks (the
// exchange of quantized payloads along graph edges / the segment all-gather of P:188, and
// the consensus rule's per-segment sum), behind one interface with two implementations:
//
//  * NCCL (one process per GPU, the production path over NVLink / NVSwitch):
//    ncclSend / ncclRecv of every plan entry in one group; ncclReduce per segment.
//  * in-process loopback (several contexts of one world inside ONE process, one host thread
//    per rank, on one GPU or on several GPUs of the box): the receiver pulls each plan entry
//    with its own cudaMemcpyAsync from the sender's payload buffer (peer copy over NVLink
//    when the ranks sit on different GPUs), after a stream wait on the sender's "payload
//    ready" event; the segment sum is a fixed-order (rank 0, 1, ...) kernel at the owner.
//    Host rendezvous (with a timeout) orders the event records before the waits.  It is the
//    single-GPU stand-in for NCCL in the tests (NCCL cannot put two ranks on one GPU) and
//    runs the same plan, buffers and graph segmentation as the NCCL path.
//
// Both are stream-ordered like NCCL: a payload buffer is not overwritten by the sender's
// next encode before every receiver has its copy.
#pragma once
#include <nccl.h>

#include <memory>
#include <vector>

#include "common.cuh"

namespace tq {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi &nccl();  // loads libnccl.so.2 on first use (fails with TQ_ENCCL if absent)

struct XferDesc {       // one payload crossing ranks in an iteration
    int slice, node, peer;
    void *buf;          // sender: the payload; receiver: where it lands
    long long bytes;
};

struct SumSeg {         // consensus rule: doubles [off, off + count) of the sum buffer, owner `root`
    long long off, count;
    int root;
};

struct Transport {
    int rank = 0, world = 1, device = 0;
    virtual ~Transport() {}
    virtual const char *name() const = 0;
    // true: every rank must take part in every exchange (the loopback's rendezvous), even with
    // an empty plan; false (NCCL point-to-point): ranks without transfers skip it
    virtual bool collective_exchange() const = 0;
    // enqueue on s every send and receive of the plan (both lists sorted by (peer, node))
    virtual void exchange(cudaStream_t s, const std::vector<XferDesc> &sends,
                          const std::vector<XferDesc> &recvs) = 0;
    // enqueue on s: for every segment, base[off..off+count) of all ranks summed onto its root
    virtual void reduce_sum(cudaStream_t s, double *base, const std::vector<SumSeg> &segs) = 0;
    // blocking: maximum of a host scalar over ranks (the stop test of tq_params.stop_tol)
    virtual double allreduce_max(double v, cudaStream_t s) = 0;
    // host rendezvous of the ranks of one process (loopback): no rank allocates device memory
    // or instantiates graphs while another rank's thread is capturing one; no-op for NCCL
    virtual void host_fence() {}
};

// id: an NCCL unique id (from tq_nccl_unique_id) or a loopback world id (tq_loopback_id)
std::unique_ptr<Transport> make_transport(const uint8_t id[128], int rank, int world, int device);
bool is_loopback_id(const uint8_t id[128]);
void new_loopback_id(uint8_t id[128]);
// tq_debug_transport_check (include/tomoq.h): every Transport operation on a synthetic plan,
// results compared with their exact host values; throws TQ_ENCCL on a mismatch
void transport_check(const uint8_t id[128], int rank, int world, int device, long long bytes, long long n_doubles,
                     int rounds);

}  // namespace tq
