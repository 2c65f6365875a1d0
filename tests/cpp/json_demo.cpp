// Test harness for the host core's JSON output (csrc/json_out.hpp and
// SelectionReport::to_json / to_csv), compared by tests/test_cli_cpu.py with the nlohmann library
// the reference is compiled against. No GPU needed.
//   json_demo numbers     stdin: one f64 bit pattern (hex) per line -> Json::number per line
//   json_demo selection   stdin: "nrec chosen" then nrec lines "k valid runs_used" + three f64
//                         bit patterns (hex), then the rationale line -> to_json, "---", to_csv
//   json_demo document    a fixed mixed document, dump(2) then dump()
#include <cstdint>
#include <cstring>
#include <iostream>
#include <string>

#include "json_out.hpp"
#include "oocnmf_b200/oocnmf.hpp"

using oocnmf::jsonout::Json;

static double from_hex(const std::string& h) {
    std::uint64_t b = std::stoull(h, nullptr, 16);
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "";
    if (mode == "numbers") {
        std::string h;
        while (std::cin >> h) std::cout << Json::number(from_hex(h)) << "\n";
        return 0;
    }
    if (mode == "selection") {
        std::size_t nrec;
        long long chosen;
        std::cin >> nrec >> chosen;
        oocnmf::SelectionReport rep;
        for (std::size_t i = 0; i < nrec; ++i) {
            oocnmf::KRecord r;
            int valid;
            std::string a, b, c;
            std::cin >> r.k >> valid >> r.runs_used >> a >> b >> c;
            r.valid = valid != 0;
            r.min_silhouette = from_hex(a), r.mean_silhouette = from_hex(b), r.mean_relative_error = from_hex(c);
            rep.records.push_back(std::move(r));
        }
        if (chosen >= 0) rep.chosen_k = oocnmf::index_t(chosen);
        std::string why;
        std::getline(std::cin >> std::ws, why);
        rep.rationale = why;
        std::cout << rep.to_json() << "\n---\n" << rep.to_csv();
        return 0;
    }
    if (mode == "document") {
        Json j;
        j["command"] = "factorize";
        j["quote \"and\" tab\t"] = "line\nbreak \\ \x01";
        j["ints"].push_back(3), j["ints"].push_back(-4);
        j["floats"].push_back(0.1), j["floats"].push_back(1e-300), j["floats"].push_back(2.0);
        j["nested"]["empty_obj"] = Json::object();
        j["nested"]["empty_arr"] = Json::array();
        j["nested"]["big"] = std::uint64_t(18446744073709551615ull);
        j["nested"]["flag"] = false;
        j["nested"]["none"] = nullptr;
        Json row;
        row["a"] = 1.5, row["b"] = "x";
        j["rows"].push_back(row), j["rows"].push_back(row);
        std::cout << j.dump(2) << "\n---\n" << j.dump() << "\n";
        return 0;
    }
    std::cerr << "usage: json_demo numbers|selection|document\n";
    return 2;
}
