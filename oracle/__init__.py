# TEST INFRASTRUCTURE: CPU oracle of the reference FTR path (see oracle.hpp).
