// connect_tcp (include/oocnmf/comm.hpp:84-87): the reference's multi-process backend. The
// reference moves every collective's payload through rank 0 over TCP sockets
// (src/comm_tcp.cpp:147-252); here TCP is only the rendezvous. Rank 0 listens on peers[0]
// ("host:port"), every other rank connects (retrying until the timeout) and says hello
// {group_id, rank}; rank 0 answers each with a fresh NCCL unique id and every rank builds an
// NCCL communicator on its GPU, so the collectives of nmf_distributed / select_k run over
// NVLink / NVSwitch like the threads backend's. Handshake errors throw CommError (ShapeError for
// malformed endpoints), with the reference's messages where the condition is the same.
#include <arpa/inet.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <sys/time.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "oocnmf_b200/oocnmf.hpp"

namespace oocnmf {
namespace {

struct Socket {
    int fd = -1;
    Socket() = default;
    explicit Socket(int f) : fd(f) {}
    Socket(const Socket&) = delete;
    Socket& operator=(const Socket&) = delete;
    Socket(Socket&& o) noexcept : fd(o.fd) { o.fd = -1; }
    Socket& operator=(Socket&& o) noexcept {
        std::swap(fd, o.fd);
        return *this;
    }
    ~Socket() {
        if (fd >= 0) ::close(fd);
    }
    bool valid() const { return fd >= 0; }
    void set_timeout(double s) const {
        timeval tv{};
        tv.tv_sec = long(s);
        tv.tv_usec = long((s - double(tv.tv_sec)) * 1e6);
        setsockopt(fd, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
        setsockopt(fd, SOL_SOCKET, SO_SNDTIMEO, &tv, sizeof tv);
    }
    void send_all(const void* p, std::size_t n) const {
        const char* c = static_cast<const char*>(p);
        while (n) {
            const ssize_t w = ::send(fd, c, n, MSG_NOSIGNAL);
            if (w <= 0) throw CommError("tcp send failed: " + std::string(std::strerror(errno)));
            c += w, n -= std::size_t(w);
        }
    }
    void recv_all(void* p, std::size_t n) const {
        char* c = static_cast<char*>(p);
        while (n) {
            const ssize_t r = ::recv(fd, c, n, 0);
            if (r == 0) throw CommError("tcp peer closed the connection");
            if (r < 0) throw CommError("tcp recv failed: " + std::string(std::strerror(errno)));
            c += r, n -= std::size_t(r);
        }
    }
};

std::pair<std::string, std::uint16_t> parse_endpoint(const std::string& ep) {
    const auto colon = ep.rfind(':');
    if (colon == std::string::npos || colon == 0 || colon + 1 == ep.size())
        throw ShapeError("endpoint must be host:port, got " + ep);
    const long port = std::strtol(ep.c_str() + colon + 1, nullptr, 10);
    if (port <= 0 || port > 65535) throw ShapeError("endpoint must be host:port, got " + ep);
    return {ep.substr(0, colon), std::uint16_t(port)};
}

sockaddr_in resolve(const std::string& host, std::uint16_t port) {
    addrinfo hints{}, *res = nullptr;
    hints.ai_family = AF_INET;
    hints.ai_socktype = SOCK_STREAM;
    if (getaddrinfo(host.c_str(), nullptr, &hints, &res) != 0 || !res)
        throw CommError("cannot resolve host: " + host);
    sockaddr_in a = *reinterpret_cast<sockaddr_in*>(res->ai_addr);
    freeaddrinfo(res);
    a.sin_port = htons(port);
    return a;
}

// This rank's GPU: OOCNMF_DEVICE, else LOCAL_RANK (torchrun / mpirun style), else rank modulo
// the visible GPUs.
int device_for(int rank) {
    if (const char* e = std::getenv("OOCNMF_DEVICE"); e && *e) return std::atoi(e);
    if (const char* e = std::getenv("LOCAL_RANK"); e && *e) return std::atoi(e);
    int count = 0;
    if (oocnmf_device_count(&count) != 0 || count < 1) throw DeviceError("connect_tcp: no CUDA device visible");
    return rank % count;
}

}  // namespace

CommHandle connect_tcp(int n, int rank, const std::vector<std::string>& peers, std::uint64_t group_id,
                       double timeout_s) {
    if (n < 1) throw ShapeError("connect_tcp: need at least one rank");
    if (rank < 0 || rank >= n) throw ShapeError("tcp rank out of range");
    if (peers.empty()) throw ShapeError("tcp backend needs endpoint addresses");
    const auto [host, port] = parse_endpoint(peers[0]);
    const int device = device_for(rank);
    CommHandle::UniqueId id{};
    if (n == 1) return CommHandle(0, 1, device, CommHandle::new_unique_id(), timeout_s);

    if (rank == 0) {
        Socket listener(::socket(AF_INET, SOCK_STREAM, 0));
        if (!listener.valid()) throw CommError("tcp socket() failed");
        const int one = 1;
        setsockopt(listener.fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
        sockaddr_in a{};
        a.sin_family = AF_INET;
        a.sin_addr.s_addr = htonl(INADDR_ANY);
        a.sin_port = htons(port);
        if (::bind(listener.fd, reinterpret_cast<sockaddr*>(&a), sizeof a) != 0)
            throw CommError("tcp bind failed on port " + std::to_string(port) + ": " + std::strerror(errno));
        if (::listen(listener.fd, n) != 0) throw CommError("tcp listen failed");
        listener.set_timeout(timeout_s);
        id = CommHandle::new_unique_id();
        std::vector<bool> seen(std::size_t(n), false);
        std::vector<Socket> conns;
        for (int got = 1; got < n; ++got) {
            Socket s(::accept(listener.fd, nullptr, nullptr));
            if (!s.valid())
                throw CommError("tcp accept timed out waiting for " + std::to_string(n - got) + " rank(s)");
            s.set_timeout(timeout_s);
            std::uint64_t hello[2];
            s.recv_all(hello, sizeof hello);
            if (hello[0] != group_id) throw CommError("tcp hello from wrong group");
            const std::uint64_t r = hello[1];
            if (r == 0 || r >= std::uint64_t(n) || seen[r])
                throw CommError("tcp hello with invalid or duplicate rank " + std::to_string(r));
            seen[r] = true;
            conns.push_back(std::move(s));
        }
        // every rank has checked in: hand out the id (NCCL's own bootstrap takes over from here)
        for (auto& s : conns) s.send_all(id.data(), id.size());
    } else {
        const sockaddr_in a = resolve(host, port);
        const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
        Socket s;
        for (;;) {
            s = Socket(::socket(AF_INET, SOCK_STREAM, 0));
            if (!s.valid()) throw CommError("tcp socket() failed");
            if (::connect(s.fd, reinterpret_cast<const sockaddr*>(&a), sizeof a) == 0) break;
            if (std::chrono::steady_clock::now() > deadline)
                throw CommError("tcp connect to " + host + ":" + std::to_string(port) + " timed out");
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
        s.set_timeout(timeout_s);
        const std::uint64_t hello[2] = {group_id, std::uint64_t(rank)};
        s.send_all(hello, sizeof hello);
        s.recv_all(id.data(), id.size());
    }
    return CommHandle(rank, n, device, id, timeout_s);
}

}  // namespace oocnmf
